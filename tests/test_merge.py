"""merge + update_neighbors.

CPU (oracle pin): the oracle's merge of the partial DTs with the border
triangulation reproduces the reference's own sequential DT (oracle/_ref,
compiled from the reference's sources; the host builder where _ref is absent)
— canonical form AND the full neighbour structure — on every instance: the
SPEC's master property on one k-way level. Plus the SPEC's merge
examples and error cases.

GPU (parity): the sm_100a merge through the C ABI against the oracle,
bit-exact (rows, order, links, parity, offsets), and the whole GPU pipeline
(assign -> find_border -> merge) against the sequential DT.
"""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_1902_07554_b200 import host

NONE = 0xFFFFFFFF


def seq_dt(points):
    """The sequential DT of all points: the reference's own (oracle/_ref) where
    built, else the host builder (pinned to it by tests/test_host.py)."""
    ids = np.arange(len(points), dtype=np.uint32)
    L = oracle.ref_lib()
    dim = points.shape[1]
    if L is None:
        t = host.triangulate(points, ids, 1)
        return t.verts, t.nbrs
    pts = np.ascontiguousarray(points, np.float64)
    h = L.ref_triangulate(dim, pts.ctypes.data_as(C.POINTER(C.c_double)), len(pts),
                          ids.ctypes.data_as(C.POINTER(C.c_uint32)), len(ids), 1)
    assert h
    try:
        S = L.ref_tri_count(h)
        v = np.empty((dim + 1, S), np.uint32)
        nb = np.empty((dim + 1, S), np.uint32)
        L.ref_tri_export(h, v.ctypes.data_as(C.POINTER(C.c_uint32)), nb.ctypes.data_as(C.POINTER(C.c_uint32)), None)
    finally:
        L.ref_tri_free(h)
    return v, nb


def canon(v):
    fin = v[:, v[-1] != NONE]
    return np.unique(np.sort(fin.T, axis=1), axis=0)


def adjacency(v, nb):
    """{row tuple: sorted tuple of neighbour row tuples} — the neighbour
    structure independent of row numbering (infinite rows included)."""
    rows = [tuple(int(x) for x in v[:, s]) for s in range(v.shape[1])]
    out = {}
    for s, r in enumerate(rows):
        out[r] = tuple(sorted(rows[t] if t != NONE else () for t in nb[:, s]))
    return out


def check_structure(v, nb):
    """Symmetric links; linked rows share exactly the facet opposite the link."""
    D1, R = v.shape
    for s in range(R):
        for d in range(D1):
            t = nb[d, s]
            assert t != NONE
            assert s in nb[:, t]
            shared = set(v[:, s]) & set(v[:, t])
            assert len(shared) == D1 - 1 and v[d, s] not in shared


CASES = [  # (dim, dist, n, k, seed)
    (2, "uniform", 4000, 4, 3),
    (3, "uniform", 4000, 4, 3),
    (2, "normal", 3000, 8, 5),
    (3, "normal", 5000, 8, 2),
    (3, "bubbles", 5000, 2, 3),
    (2, "lines", 4000, 4, 7),
]

_inst = {}


def instance(case):
    if case not in _inst:
        dim, dist, n, k, seed = case
        inst = host.make_instance(dict(name="m", dist=dist, dim=dim, n=n, seed=seed, frac=0.02, k=k))
        lab = oracle.assign_kdtree(inst.points, inst.sample_ids, inst.sample_labels)
        P = host.build_partials(inst.points, lab, k, 1)
        fb = oracle.find_border(inst.points, lab, P)
        _inst[case] = (inst.points, lab, P, fb)
    return _inst[case]


def border_tri(points, vids):
    if len(vids) < points.shape[1] + 1:
        D1 = points.shape[1] + 1
        return host.Tri(np.zeros((D1, 0), np.uint32), np.zeros((D1, 0), np.uint32), np.zeros(0, np.int8))
    return host.triangulate(points, vids, 7)


def merge_inputs(case, which):
    pts, lab, P, fb = instance(case)
    flags = fb["border"] if which == "bfs" else fb["positive"]
    vids = fb["vertices_border"] if which == "bfs" else fb["vertices_positive"]
    return pts, lab, P, flags, border_tri(pts, vids)


# ---------------------------------------------------------------- CPU: oracle pin
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("which", ["bfs", "positive"])
def test_oracle_merge_equals_sequential_dt(case, which):
    pts, lab, P, flags, tb = merge_inputs(case, which)
    v, nb, par, off = oracle.merge(P, flags, tb, lab)
    sv, snb = seq_dt(pts)
    assert np.array_equal(canon(v), canon(sv))
    check_structure(v, nb)
    assert adjacency(v, nb) == adjacency(sv, snb)
    fin = v[-1] != NONE
    assert np.all(par[fin] != 0) and np.all(par[~fin] == 0)
    k = P.k
    assert off[k + 2] == v.shape[1] and off[k + 1] == fin.sum() and np.all(np.diff(off.astype(np.int64)) >= 0)
    # kept rows of part p carry part p's vertices; inserted rows come from T_B
    for p in range(k):
        rows = v[:, off[p]:off[p + 1]]
        assert np.all(lab[rows] == p)


def test_oracle_merge_empty_border_is_disjoint_union():
    """empty border, empty T_B -> T = disjoint union of partials."""
    pts, lab, P, fb = instance(CASES[0])
    D1 = P.verts.shape[0]
    empty = host.Tri(np.zeros((D1, 0), np.uint32), np.zeros((D1, 0), np.uint32), np.zeros(0, np.int8))
    v, nb, par, off = oracle.merge(P, np.zeros(P.S, np.uint8), empty, lab, hull=False)
    fin = P.verts[-1] != NONE
    assert v.shape[1] == fin.sum()
    assert np.array_equal(v, P.verts[:, fin])
    assert np.array_equal(par, P.parity[fin])


def test_oracle_merge_k1_identity():
    """k = 1: no border; the merge re-derives the partial's own hull."""
    pts = host.generate("uniform", 3, 2000, 11)
    lab = np.zeros(len(pts), np.uint32)
    P = host.build_partials(pts, lab, 1, 1)
    D1 = 4
    empty = host.Tri(np.zeros((D1, 0), np.uint32), np.zeros((D1, 0), np.uint32), np.zeros(0, np.int8))
    v, nb, par, off = oracle.merge(P, np.zeros(P.S, np.uint8), empty, lab)
    assert adjacency(v, nb) == adjacency(P.verts, P.nbrs)


def test_oracle_merge_rule_ii_negative():
    """a single-partition T_B simplex absent from B is excluded."""
    pts, lab, P, flags, tb = merge_inputs(CASES[1], "bfs")
    v, nb, par, off = oracle.merge(P, flags, tb, lab, hull=False)
    k = P.k
    ins = v[:, off[k]:off[k + 1]]
    single = np.all(lab[ins] == lab[ins[0]], axis=0)
    btup = {tuple(P.verts[:, s]) for s in np.nonzero(flags)[0] if P.verts[-1, s] != NONE}
    for s in np.nonzero(single)[0]:
        assert tuple(ins[:, s]) in btup
    # and every excluded finite single-partition T_B row is absent from B
    tin = {tuple(ins[:, s]) for s in range(ins.shape[1])}
    for t in range(tb.verts.shape[1]):
        r = tuple(tb.verts[:, t])
        if r[-1] != NONE and r not in tin:
            assert len(set(lab[list(r)])) == 1 and r not in btup


def test_oracle_merge_two_distant_clusters():
    """unit boxes at the origin and (10,10), k = 2: the merge adds
    the cross-cluster simplices covering the hull gap."""
    rng = np.random.default_rng(4)
    a = rng.random((1500, 2))
    b = rng.random((1500, 2)) + 10.0
    pts = np.concatenate([a, b])
    lab = np.repeat(np.arange(2, dtype=np.uint32), 1500)
    P = host.build_partials(pts, lab, 2, 1)
    fb = oracle.find_border(pts, lab, P, "exact")
    tb = border_tri(pts, fb["vertices_border"])
    v, nb, par, off = oracle.merge(P, fb["border"], tb, lab)
    sv, snb = seq_dt(pts)
    assert np.array_equal(canon(v), canon(sv))
    fin = v[:, v[-1] != NONE]
    assert np.any(np.any(lab[fin] != lab[fin[0]], axis=0))


def test_oracle_merge_inconsistent():
    """a simplex inserted twice is InconsistentMerge."""
    pts, lab, P, flags, tb = merge_inputs(CASES[0], "positive")
    SB = tb.verts.shape[1]
    dup = host.Tri(np.concatenate([tb.verts, tb.verts], axis=1),
                   np.concatenate([tb.nbrs, np.where(tb.nbrs == NONE, NONE, tb.nbrs + SB)], axis=1).astype(np.uint32),
                   np.concatenate([tb.parity, tb.parity]))
    with pytest.raises(RuntimeError, match="InconsistentMerge"):
        oracle.merge(P, flags, dup, lab)


# ---------------------------------------------------------------- GPU parity
def gpu_case(ctx, case, which, hull=True):
    from paper_1902_07554_b200 import gpu
    pts, lab, P, flags, tb = merge_inputs(case, which)
    g = gpu.merge(P, flags, tb, lab, hull=hull, ctx=ctx)
    o = oracle.merge(P, flags, tb, lab, hull=hull)
    return g, o


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("which", ["bfs", "positive"])
def test_gpu_merge_bit_exact(ctx, case, which):
    g, (v, nb, par, off) = gpu_case(ctx, case, which)
    assert np.array_equal(g.offsets, off)
    assert np.array_equal(g.verts, v)
    assert np.array_equal(g.parity, par)
    assert np.array_equal(g.nbrs, nb)


@pytest.mark.gpu
def test_gpu_merge_without_hull(ctx):
    g, (v, nb, par, off) = gpu_case(ctx, CASES[1], "bfs", hull=False)
    assert np.array_equal(g.verts, v) and np.array_equal(g.nbrs, nb) and np.array_equal(g.offsets, off)
    assert np.any(g.nbrs == NONE)


@pytest.mark.gpu
def test_gpu_merge_edge_cases(ctx):
    from paper_1902_07554_b200 import gpu
    pts, lab, P, fb = instance(CASES[0])
    D1 = P.verts.shape[0]
    empty = host.Tri(np.zeros((D1, 0), np.uint32), np.zeros((D1, 0), np.uint32), np.zeros(0, np.int8))
    zero = np.zeros(P.S, np.uint8)
    for hull in (False, True):
        g = gpu.merge(P, zero, empty, lab, hull=hull, ctx=ctx)
        v, nb, par, off = oracle.merge(P, zero, empty, lab, hull=hull)
        assert np.array_equal(g.verts, v) and np.array_equal(g.nbrs, nb) and np.array_equal(g.offsets, off)
    # every row a border row, T_B = the whole DT: the merge is T_B itself
    allb = np.ones(P.S, np.uint8)
    tb = host.triangulate(pts, np.arange(len(pts), dtype=np.uint32), 3)
    g = gpu.merge(P, allb, tb, lab, ctx=ctx)
    v, nb, par, off = oracle.merge(P, allb, tb, lab)
    assert np.array_equal(g.verts, v) and np.array_equal(g.nbrs, nb)
    assert adjacency(g.verts, g.nbrs) == adjacency(tb.verts, tb.nbrs)
    # k = 1
    pk = host.build_partials(pts, np.zeros(len(pts), np.uint32), 1, 1)
    g = gpu.merge(pk, np.zeros(pk.S, np.uint8), empty, np.zeros(len(pts), np.uint32), ctx=ctx)
    assert adjacency(g.verts, g.nbrs) == adjacency(pk.verts, pk.nbrs)


@pytest.mark.gpu
def test_gpu_merge_inconsistent(ctx):
    from paper_1902_07554_b200 import gpu
    pts, lab, P, flags, tb = merge_inputs(CASES[0], "positive")
    SB = tb.verts.shape[1]
    dup = host.Tri(np.concatenate([tb.verts, tb.verts], axis=1),
                   np.concatenate([tb.nbrs, np.where(tb.nbrs == NONE, NONE, tb.nbrs + SB)], axis=1).astype(np.uint32),
                   np.concatenate([tb.parity, tb.parity]))
    with pytest.raises(gpu.InconsistentMerge):
        gpu.merge(P, flags, dup, lab, ctx=ctx)
    # the context stays usable
    g, (v, nb, par, off) = gpu_case(ctx, CASES[0], "positive")
    assert np.array_equal(g.nbrs, nb)


@pytest.mark.gpu
@pytest.mark.parametrize("dim,dist,n,k", [(3, "uniform", 60_000, 16), (2, "normal", 60_000, 8),
                                          (3, "bubbles", 60_000, 8)])
@pytest.mark.parametrize("which", ["bfs", "positive"])
def test_gpu_pipeline_equals_sequential_dt(ctx, dim, dist, n, k, which):
    """assign_points -> find_border -> merge, all on the GPU (host partial and
    border DTs): the master property of SPEC.md:516 on one k-way level."""
    from paper_1902_07554_b200 import dc
    pts = host.deduplicate(host.generate(dist, dim, n, 9))
    r = dc.delaunay_dc_once(pts, k, seed=9, border=which, ctx=ctx)
    sv, snb = seq_dt(pts)
    assert np.array_equal(canon(r.merged.verts), canon(sv))
    assert adjacency(r.merged.verts, r.merged.nbrs) == adjacency(sv, snb)


def ring_instance():
    """2-D points near a circle: nearly every point is a hull vertex, so the
    merged hull has more facets than the GPU's single-CTA sort takes (16384)."""
    if "ring" not in _inst:
        rng = np.random.default_rng(12)
        n = 20_000
        th = np.sort(rng.random(n)) * 2 * np.pi
        r = 1.0 - 1e-11 * rng.random(n)
        pts = np.stack([r * np.cos(th), r * np.sin(th)], axis=1)
        lab = (np.arange(n) * 4 // n).astype(np.uint32)  # 4 arcs
        P = host.build_partials(pts, lab, 4, 1)
        fb = oracle.find_border(pts, lab, P)
        _inst["ring"] = (pts, lab, P, fb)
    return _inst["ring"]


def test_oracle_merge_many_hull_facets():
    pts, lab, P, fb = ring_instance()
    tb = border_tri(pts, fb["vertices_border"])
    v, nb, par, off = oracle.merge(P, fb["border"], tb, lab)
    sv, snb = seq_dt(pts)
    assert np.array_equal(canon(v), canon(sv))
    assert v.shape[1] - off[P.k + 1] > 16384


@pytest.mark.gpu
def test_gpu_merge_many_hull_facets(ctx):
    from paper_1902_07554_b200 import gpu
    pts, lab, P, fb = ring_instance()
    tb = border_tri(pts, fb["vertices_border"])
    g = gpu.merge(P, fb["border"], tb, lab, ctx=ctx)
    v, nb, par, off = oracle.merge(P, fb["border"], tb, lab)
    assert np.array_equal(g.offsets, off)
    assert np.array_equal(g.verts, v) and np.array_equal(g.nbrs, nb) and np.array_equal(g.parity, par)
