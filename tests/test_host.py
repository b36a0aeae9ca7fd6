"""Host setup (not on the measured path, but it produces the inputs both the
GPU and the oracle consume): DT builder == reference triangulate_seq
canonical forms (golden, from the reference's compiled code), SPEC
partitioner contract, generator determinism, dedup and sampling."""
import os

import numpy as np
import pytest

from paper_1902_07554_b200 import host

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def canon(tri: host.Tri) -> np.ndarray:
    v = tri.verts
    fin = v[:, v[-1] != 0xFFFFFFFF]
    return np.unique(np.sort(fin.T, axis=1), axis=0)


@pytest.fixture(scope="module")
def dtg():
    return np.load(os.path.join(GOLDEN, "dt_canon.npz"))


@pytest.mark.parametrize("key", ["d2_0", "d2_1", "d2_2", "d3_0", "d3_1", "d3_2", "bubbles", "lines"])
def test_dt_matches_reference_canonical(dtg, key):
    pts = dtg[f"{key}_pts"]
    ref = dtg[f"{key}_canon"]
    for seed in (1, 99):
        tri = host.triangulate(pts, np.arange(len(pts), dtype=np.uint32), seed)
        assert np.array_equal(canon(tri), ref)


def test_dt_structure_invariants():
    pts = host.generate("uniform", 3, 3000, 5)
    tri = host.triangulate(pts, np.arange(3000, dtype=np.uint32), 3)
    v, nb, par = tri.verts, tri.nbrs, tri.parity
    S = v.shape[1]
    fin = v[-1] != 0xFFFFFFFF
    assert np.all(par[fin] != 0) and np.all(par[~fin] == 0)
    assert np.all(np.diff(v.astype(np.int64), axis=0) > 0)  # ascending, infinite last
    # neighbour symmetry and facet sharing (D shared vertices)
    for s in range(0, S, 7):
        for d in range(4):
            t = nb[d, s]
            assert s in nb[:, t]
            assert len(set(v[:, s]) & set(v[:, t])) == 3
    # finite simplices per point in [6, 8] (SPEC acceptance 8, desk scale)
    assert 5.5 <= fin.sum() / 3000 <= 8.0


def test_sequential_dt_spec_examples():
    pts = np.array([[0, 0], [1, 0], [0, 1]], np.float64)
    assert np.array_equal(canon(host.triangulate(pts, np.arange(3, dtype=np.uint32), 1)), [[0, 1, 2]])
    pts = np.array([[0, 0], [1, 0], [0, 1], [2, 2]], np.float64)
    assert np.array_equal(canon(host.triangulate(pts, np.arange(4, dtype=np.uint32), 1)), [[0, 1, 2], [1, 2, 3]])
    with pytest.raises(ValueError):
        host.triangulate(np.array([[i, 2.0 * i] for i in range(5)], np.float64), np.arange(5, dtype=np.uint32), 1)


def _csr(edges, n):
    adj = [[] for _ in range(n)]
    for a, b, w in edges:
        adj[a].append((b, w))
        adj[b].append((a, w))
    xadj = np.zeros(n + 1, np.uint32)
    for i in range(n):
        xadj[i + 1] = xadj[i] + len(adj[i])
    return xadj, np.array([b for l in adj for b, _ in l], np.uint32), np.array([w for l in adj for _, w in l], np.int32)


def test_partitioner_spec_examples():
    # path v0-v1-v2-v3 weights (10,1,10), k=2 -> {v0,v1 | v2,v3}, cut 1
    lab, cut = host.partition_csr(*_csr([(0, 1, 10), (1, 2, 1), (2, 3, 10)], 4), k=2)
    assert cut == 1 and lab[0] == lab[1] and lab[2] == lab[3] and lab[0] != lab[2]
    # k=1 -> all 0, cut 0
    lab, cut = host.partition_csr(*_csr([(0, 1, 10), (1, 2, 1), (2, 3, 10)], 4), k=1)
    assert cut == 0 and not lab.any()
    # K4 unit weights, k=2 -> 2/2 split, cut 4
    lab, cut = host.partition_csr(*_csr([(a, b, 1) for a in range(4) for b in range(a + 1, 4)], 4), k=2)
    assert cut == 4 and np.bincount(lab).tolist() == [2, 2]


@pytest.mark.parametrize("k", [2, 4, 8, 16])
def test_partitioner_balance(k):
    pts = host.generate("uniform", 2, 3000, 17)
    sid = np.arange(3000, dtype=np.uint32)
    lab, cut = host.partition_sample(pts, sid, k, seed=3)
    sizes = np.bincount(lab, minlength=k)
    assert sizes.min() > 0
    assert sizes.max() <= (1.05) * np.ceil(3000 / k)  # SPEC.md:252 balance constraint


def test_generators_deterministic_and_bounded():
    for dist, dim in (("uniform", 2), ("uniform", 3), ("normal", 3), ("bubbles", 3), ("lines", 2)):
        a = host.generate(dist, dim, 5000, 9)
        b = host.generate(dist, dim, 5000, 9)
        c = host.generate(dist, dim, 5000, 10)
        assert np.array_equal(a, b) and not np.array_equal(a, c)
        assert np.isfinite(a).all()
    u = host.generate("uniform", 3, 5000, 1)
    assert u.min() >= 0 and u.max() < 1


def test_dedup_and_sample():
    pts = np.array([[0.5, 0.25], [0.75, 0.125], [0.5, 0.25]], np.float64)
    d = host.deduplicate(pts)
    assert len(d) == 2 and np.array_equal(d[0], pts[0]) and np.array_equal(d[1], pts[1])
    s1 = host.draw_sample(10000, 100, 5)
    s2 = host.draw_sample(10000, 100, 5)
    assert np.array_equal(s1, s2) and len(np.unique(s1)) == 100 and s1.max() < 10000


def test_partials_cover_every_point_once():
    inst = host.make_instance(1, n=5000, k=4, frac=0.02)
    import oracle
    lab = oracle.assign_kdtree(inst.points, inst.sample_ids, inst.sample_labels)
    part = host.attach_partials(inst, lab)
    for p in range(4):
        lo, hi = part.offsets[p], part.offsets[p + 1]
        v = part.verts[:, lo:hi]
        ids = np.unique(v[v != 0xFFFFFFFF])
        assert np.array_equal(ids, np.nonzero(lab == p)[0])


def _rows(tri):
    """Row set with each row's neighbours as vertex tuples (order-independent form)."""
    v, nb = tri.verts, tri.nbrs
    key = [tuple(v[:, s]) for s in range(v.shape[1])]
    return {key[s]: (tri.parity[s], frozenset(key[nb[d, s]] for d in range(v.shape[0]))) for s in range(v.shape[1])}


@pytest.mark.parametrize("dim", [2, 3])
def test_row_order_morton_vs_slot(dim, monkeypatch):
    """compact() emits rows along a Morton curve (default) or in slot order
    (SBDT_HOST_ROW_ORDER=slot): the same triangulation either way (rows,
    parities, neighbour links), and the Morton order is the spatially coherent
    one (fewer distinct vertices per 32 consecutive rows)."""
    pts = host.generate("uniform", dim, 20000, 11)
    ids = np.arange(20000, dtype=np.uint32)
    monkeypatch.delenv("SBDT_HOST_ROW_ORDER", raising=False)
    tm = host.triangulate(pts, ids, 7)
    monkeypatch.setenv("SBDT_HOST_ROW_ORDER", "slot")
    ts = host.triangulate(pts, ids, 7)
    assert tm.verts.shape == ts.verts.shape
    assert _rows(tm) == _rows(ts)
    assert not np.array_equal(tm.verts, ts.verts)

    def distinct(t):
        g = t.verts.shape[1] // 32
        blocks = t.verts[:, :g * 32].reshape(dim + 1, g, 32)
        return np.mean([len(np.unique(blocks[:, i, :])) for i in range(0, g, 5)])

    assert distinct(tm) < 0.7 * distinct(ts)
