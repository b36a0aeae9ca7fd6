"""The CPU oracle, pinned: SPEC.md known-answer examples, the reference's own
primitive test cases (proj/tests/test_geometry.cpp), and golden vectors
produced by the reference's compiled code (tests/golden/, make_golden.py).
Also: if oracle/_ref is present (this container), the restatement is checked
live against the reference instantiation on fresh random instances."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle
from paper_1902_07554_b200 import host

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
P = oracle._p
L = oracle.lib()


def orient(pts):
    a = np.ascontiguousarray(np.asarray(pts, np.float64).ravel())
    return L.oracle_orient(len(pts[0]), P(a, C.c_double))


def in_sphere(pts, q):
    a = np.ascontiguousarray(np.asarray(pts, np.float64).ravel())
    qq = np.ascontiguousarray(np.asarray(q, np.float64))
    return L.oracle_in_sphere(len(q), P(a, C.c_double), P(qq, C.c_double))


def circumsphere(pts):
    dim = len(pts[0])
    a = np.ascontiguousarray(np.asarray(pts, np.float64).ravel())
    out = np.zeros(dim + 1)
    st = L.oracle_circumsphere(dim, P(a, C.c_double), P(out, C.c_double))
    return st, out


def box_sphere(lo, hi, c, r2):
    lo, hi, c = (np.ascontiguousarray(np.asarray(v, np.float64)) for v in (lo, hi, c))
    return L.oracle_box_sphere(len(lo), P(lo, C.c_double), P(hi, C.c_double), P(c, C.c_double), float(r2))


def halfspace(facet, inner, lo, hi):
    f = np.ascontiguousarray(np.asarray(facet, np.float64).ravel())
    i, lo, hi = (np.ascontiguousarray(np.asarray(v, np.float64)) for v in (inner, lo, hi))
    return L.oracle_halfspace_box(len(lo), P(f, C.c_double), P(i, C.c_double), P(lo, C.c_double), P(hi, C.c_double))


# ---- SPEC.md geometry examples and test_geometry.cpp:13-119
def test_orient_kats():
    assert orient([(0, 0), (1, 0), (0, 1)]) == 1
    assert orient([(0, 0), (1, 0), (2, 0)]) == 0
    assert orient([(0, 0), (0, 1), (1, 0)]) == -1
    assert orient([(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]) == 1
    assert orient([(0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0)]) == 0
    assert orient([(0, 0, 0), (0, 1, 0), (1, 0, 0), (0, 0, 1)]) == -1


def test_in_sphere_kats():
    t = [(0, 0), (2, 0), (0, 2)]
    assert in_sphere(t, (1, 1)) == 1
    assert in_sphere(t, (2, 2)) == 0
    assert in_sphere(t, (5, 5)) == -1
    t3 = [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]
    assert in_sphere(t3, (0.5, 0.5, 0.5)) == 1
    assert in_sphere(t3, (1, 1, 1)) == 0
    assert in_sphere(t3, (2, 2, 2)) == -1


def test_circumsphere_kats():
    st, s = circumsphere([(0, 0), (2, 0), (0, 2)])
    assert st == 0 and np.allclose(s, [1, 1, 2])
    st, s = circumsphere([(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)])
    assert st == 0 and np.allclose(s, [0.5, 0.5, 0.5, 0.75])
    st, _ = circumsphere([(0, 0), (1, 0), (2, 0)])
    assert st == 1  # DegenerateSimplex


def test_box_sphere_kats():
    assert box_sphere((0, 0, 0), (1, 1, 1), (0.5, 0.5, 0.5), 0.01)
    assert not box_sphere((0, 0, 0), (1, 1, 1), (2, 0, 0), 0.25)
    assert box_sphere((0, 0, 0), (1, 1, 1), (1.2, 0.5, 0.5), 0.09)


def test_halfspace_kats():
    f = [(0, 0), (0, 1)]
    inner = (-1, 0.5)
    assert halfspace(f, inner, (1, 0), (2, 1))
    assert not halfspace(f, inner, (-2, 0), (-1, 1))
    assert halfspace(f, inner, (-0.5, -0.5), (0.5, 0.5))
    assert not halfspace(f, inner, (-1, 0), (0, 1))  # touching is not outside


# ---- golden vectors from the reference's compiled geometry.cpp
@pytest.fixture(scope="module")
def prim():
    return np.load(os.path.join(GOLDEN, "primitives.npz"))


@pytest.mark.parametrize("dim", [2, 3])
def test_orient_golden(prim, dim):
    pts, out = prim[f"orient{dim}_pts"], prim[f"orient{dim}_out"]
    got = np.array([L.oracle_orient(dim, P(np.ascontiguousarray(p), C.c_double)) for p in pts])
    assert np.array_equal(got, out)
    assert (out == 0).sum() + (out != 0).sum() == len(out)


@pytest.mark.parametrize("dim", [2, 3])
def test_in_sphere_golden(prim, dim):
    pts, q, out = prim[f"insphere{dim}_pts"], prim[f"insphere{dim}_q"], prim[f"insphere{dim}_out"]
    got = np.array([L.oracle_in_sphere(dim, P(np.ascontiguousarray(p), C.c_double),
                                       P(np.ascontiguousarray(qq), C.c_double)) for p, qq in zip(pts, q)])
    assert np.array_equal(got, out)


@pytest.mark.parametrize("dim", [2, 3])
def test_circumsphere_golden_bit_exact(prim, dim):
    pts, out, st = prim[f"circum{dim}_pts"], prim[f"circum{dim}_out"], prim[f"circum{dim}_status"]
    for p, o, s in zip(pts, out, st):
        s2, o2 = circumsphere(p.reshape(dim + 1, dim))
        assert s2 == s
        if s == 0:
            assert np.array_equal(o2, o)


@pytest.mark.parametrize("dim", [2, 3])
def test_box_sphere_golden(prim, dim):
    rows, out = prim[f"boxsphere{dim}"], prim[f"boxsphere{dim}_out"]
    got = [box_sphere(r[:dim], r[dim:2 * dim], r[2 * dim:3 * dim], r[3 * dim]) for r in rows]
    assert np.array_equal(np.array(got, np.int8), out)


@pytest.mark.parametrize("dim", [2, 3])
def test_halfspace_golden(prim, dim):
    rows, out = prim[f"halfspace{dim}"], prim[f"halfspace{dim}_out"]
    for r, o in zip(rows, out):
        if o < 0:
            continue
        f = r[:dim * dim].reshape(dim, dim)
        i = r[dim * dim:dim * dim + dim]
        lo, hi = r[dim * dim + dim:dim * dim + 2 * dim], r[dim * dim + 2 * dim:]
        assert halfspace(f, i, lo, hi) == o


# ---- assign_points SPEC examples
def test_assign_kats():
    pts = np.array([[0, 0], [1, 0], [0.2, 0.1], [0.5, 0.0]], np.float64)
    sid = np.array([0, 1], np.uint32)
    slab = np.array([0, 1], np.uint32)
    for fn in (oracle.assign_brute, oracle.assign_kdtree):
        lab = fn(pts, sid, slab)
        assert lab[2] == 0  # nearer to (0,0)
        assert lab[3] == 0  # equidistant -> lowest sample id
    # tie toward the lowest sample PointId, not the first listed sample
    lab = oracle.assign_brute(pts, np.array([1, 0], np.uint32), np.array([7, 3], np.uint32))
    assert lab[3] == 3


def test_assign_lattice_ties_kdtree_equals_brute():
    g = np.stack(np.meshgrid(np.arange(30.0), np.arange(30.0)), -1).reshape(-1, 2)
    rng = np.random.default_rng(3)
    sid = np.sort(rng.choice(len(g), 60, replace=False)).astype(np.uint32)
    slab = rng.integers(0, 5, 60).astype(np.uint32)
    q = np.vstack([g, g + 0.5])  # many exact ties on the lattice
    pts = np.vstack([g, q[len(g):]])
    a = oracle.assign_brute(pts, sid, slab)
    b = oracle.assign_kdtree(pts, sid, slab)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("dim", [2, 3])
def test_assign_kdtree_equals_brute_random(dim):
    pts = host.generate("uniform", dim, 20000, 11)
    sid = host.draw_sample(len(pts), 300, 11)
    slab = (np.arange(300) % 7).astype(np.uint32)
    assert np.array_equal(oracle.assign_brute(pts, sid, slab), oracle.assign_kdtree(pts, sid, slab))


# ---- path golden fixtures (reference-primitive instantiation)
@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_path_golden(cfg):
    z = np.load(os.path.join(GOLDEN, f"path_cfg{cfg}.npz"))
    pts, lab = z["points"], z["labels"]
    assert np.array_equal(oracle.assign_brute(pts, z["sample_ids"], z["sample_labels"]), lab)
    assert np.array_equal(oracle.assign_kdtree(pts, z["sample_ids"], z["sample_labels"]), lab)
    part = host.Partials(z["offsets"], z["verts"], z["nbrs"], z["parity"])
    sets = {}
    for pol in ("bbox", "grid", "exact"):
        o = oracle.find_border(pts, lab, part, pol)
        assert np.array_equal(np.packbits(o["positive"]), z[f"{pol}_positive"])
        assert np.array_equal(np.packbits(o["border"]), z[f"{pol}_border"])
        assert np.array_equal(o["vertices_positive"], z[f"{pol}_vpos"])
        assert np.array_equal(o["vertices_border"], z[f"{pol}_vbfs"])
        sets[pol] = set(o["vertices_border"].tolist())
    # SPEC.md:445,519 monotone chain exact <= grid <= bbox
    assert sets["exact"] <= sets["grid"] <= sets["bbox"]


def test_find_border_k1_empty():
    inst = host.make_instance(1, n=3000, k=1, frac=0.02)
    lab = np.zeros(inst.n, np.uint32)
    part = host.attach_partials(inst, lab)
    for pol in ("bbox", "grid", "exact"):
        o = oracle.find_border(inst.points, lab, part, pol)
        assert o["positive"].sum() == 0 and len(o["vertices_border"]) == 0


def test_two_distant_clusters_hull_rule():
    # two distant clusters -> only hull-facing simplices border
    rng = np.random.default_rng(5)
    a = rng.random((400, 2))
    b = rng.random((400, 2)) + np.array([10.0, 10.0])
    pts = np.vstack([a, b])
    lab = np.r_[np.zeros(400), np.ones(400)].astype(np.uint32)
    part = host.build_partials(pts, lab, 2, 1)
    o = oracle.find_border(pts, lab, part, "grid")
    inf = part.verts[-1] == 0xFFFFFFFF
    assert o["border"].sum() > 0
    assert o["border"][inf].sum() > 0  # infinite simplices face the other cluster
    g = oracle.find_border(pts, lab, part, "exact")
    assert set(g["vertices_border"]) <= set(o["vertices_border"])


@pytest.mark.skipif(oracle.ref_lib() is None, reason="oracle/_ref not built (no /root/reference)")
@pytest.mark.parametrize("cfg", [2, 4])
def test_oracle_equals_reference_instantiation_live(cfg):
    R = oracle.ref_lib()
    inst = host.make_instance(cfg, n=15000, k=6, frac=0.02, seed=77)
    lab = oracle.assign_kdtree(inst.points, inst.sample_ids, inst.sample_labels)
    part = host.attach_partials(inst, lab)
    pts = np.ascontiguousarray(inst.points)
    for pol, code in (("grid", 1), ("exact", 2)):
        o = oracle.find_border(pts, lab, part, pol)
        pos, bor = np.empty(part.S, np.uint8), np.empty(part.S, np.uint8)
        vp, vb = np.empty(inst.n, np.uint32), np.empty(inst.n, np.uint32)
        a, b = C.c_uint64(), C.c_uint64()
        R.ref_find_border(inst.dim, P(pts, C.c_double), inst.n, P(lab, C.c_uint32), part.k, P(part.offsets, C.c_uint64),
                          P(part.verts, C.c_uint32), P(part.nbrs, C.c_uint32), P(part.parity, C.c_int8), code, 1.0,
                          P(pos, C.c_uint8), P(bor, C.c_uint8), P(vp, C.c_uint32), C.byref(a), P(vb, C.c_uint32),
                          C.byref(b))
        assert np.array_equal(o["positive"], pos)
        assert np.array_equal(o["border"], bor)
        assert np.array_equal(o["vertices_border"], vb[:b.value])
