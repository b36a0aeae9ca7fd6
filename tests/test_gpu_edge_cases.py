"""GPU parity on the edge cases the reference's contract names (SPEC.md
acceptance criteria): exact ties and cospherical / collinear
configurations (integer lattices), tiny inputs, a part without points, and a
far-from-origin translate (binning and prefilter bounds under large |x|).
Every case is compared bit for bit with the CPU oracle through the C ABI."""
import numpy as np
import pytest

import oracle
from paper_1902_07554_b200 import gpu, host

pytestmark = pytest.mark.gpu


def _check(points, sample_ids, sample_labels, k, ctx, seed=7, policies=("grid", "bbox", "exact")):
    part = gpu.assign_points(points, sample_ids, sample_labels, k, ctx=ctx)
    ref = oracle.assign_brute(points, sample_ids, sample_labels)
    assert np.array_equal(part.labels, ref)
    partials = host.build_partials(points, ref, k, seed)
    for policy in policies:
        g = gpu.find_border(points, ref, partials, gpu.IntersectionPolicy(policy, 1.0), hull_bfs=True, ctx=ctx)
        o = oracle.find_border(points, ref, partials, policy)
        assert np.array_equal(g.positive, o["positive"]), policy
        assert np.array_equal(g.border, o["border"]), policy
        assert np.array_equal(g.positive_vertex_ids, o["vertices_positive"]), policy
        assert np.array_equal(g.border_vertex_ids, o["vertices_border"]), policy
    return part, partials


def _lattice(dim, side, jitter=0.0, seed=0):
    axes = [np.arange(side, dtype=np.float64)] * dim
    pts = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, dim)
    if jitter:
        pts = pts + np.random.default_rng(seed).uniform(-jitter, jitter, pts.shape)
    return np.ascontiguousarray(pts)


@pytest.mark.parametrize("dim,side", [(2, 300), (3, 40)])
def test_integer_lattice_assignment_ties(dim, side, ctx):
    """Exact lattice: equidistant samples everywhere; the lowest sample
    PointId must win (assign_points only: the reference's DT rejects exact
    lattices as affinely degenerate beyond its tie-break)."""
    pts = _lattice(dim, side)
    rng = np.random.default_rng(1)
    sid = np.sort(rng.choice(len(pts), size=len(pts) // 20, replace=False)).astype(np.uint32)
    slab = (np.arange(len(sid)) % 7).astype(np.uint32)
    part = gpu.assign_points(pts, sid, slab, 7, ctx=ctx)
    assert np.array_equal(part.labels, oracle.assign_brute(pts, sid, slab))


@pytest.mark.parametrize("dim,side", [(2, 60), (3, 16)])
def test_jittered_lattice(dim, side, ctx):
    """Lattice + 1e-7 jitter: near-cospherical simplices everywhere."""
    pts = _lattice(dim, side, jitter=1e-7, seed=dim)
    rng = np.random.default_rng(1)
    sid = np.sort(rng.choice(len(pts), size=len(pts) // 20, replace=False)).astype(np.uint32)
    slab = np.minimum((pts[sid, 0] * 4 // side).astype(np.uint32), 3)
    _check(pts, sid, slab, 4, ctx)


def test_tiny_inputs(ctx):
    rng = np.random.default_rng(3)
    pts = np.ascontiguousarray(rng.random((40, 2)))
    sid = np.array([0, 5, 11, 17, 23, 31], np.uint32)
    slab = np.array([0, 0, 1, 1, 0, 1], np.uint32)
    _check(pts, sid, slab, 2, ctx)
    pts3 = np.ascontiguousarray(rng.random((60, 3)))
    sid3 = np.array([1, 7, 13, 29, 41, 50, 55], np.uint32)
    slab3 = np.array([0, 1, 2, 0, 1, 2, 0], np.uint32)
    _check(pts3, sid3, slab3, 3, ctx)


def test_part_without_points(ctx):
    """k = 5 but no sample carries label 4: part 4 is empty (no points, no
    simplex rows; the DT builder needs >= D+1 points, so its empty row range
    is appended) and must be handled by the part offsets and the grid."""
    inst = host.make_instance(1, n=30_000, k=4)
    part = gpu.assign_points(inst.points, inst.sample_ids, inst.sample_labels, 5, ctx=ctx)
    ref = oracle.assign_brute(inst.points, inst.sample_ids, inst.sample_labels)
    assert np.array_equal(part.labels, ref)
    assert part.parts_offsets[4] == part.parts_offsets[5] == len(ref)
    p4 = host.build_partials(inst.points, ref, 4, 7)
    p5 = host.Partials(np.append(p4.offsets, p4.offsets[-1]).astype(np.uint64), p4.verts, p4.nbrs, p4.parity)
    for policy in ("grid", "bbox", "exact"):
        g = gpu.find_border(inst.points, ref, p5, gpu.IntersectionPolicy(policy, 1.0), hull_bfs=True, ctx=ctx)
        g4 = gpu.find_border(inst.points, ref, p4, gpu.IntersectionPolicy(policy, 1.0), hull_bfs=True, ctx=ctx)
        o = oracle.find_border(inst.points, ref, p4, policy)
        assert np.array_equal(g.positive, o["positive"]) and np.array_equal(g4.positive, o["positive"])
        assert np.array_equal(g.border, o["border"])
        assert np.array_equal(g.positive_vertex_ids, o["vertices_positive"])


@pytest.mark.parametrize("shift", [1e3, -2.5e5])
def test_far_from_origin(shift, ctx):
    """A translated instance: the grid origin, the packed prefilter offsets and
    every margin are relative to large |x|."""
    inst = host.make_instance(2, n=40_000, k=8)
    pts = np.ascontiguousarray(inst.points + shift)
    _check(pts, inst.sample_ids, inst.sample_labels, 8, ctx, policies=("grid", "exact"))


def test_jittered_lattice_near_degenerate(ctx):
    """Lattice plus 1e-9 jitter: binary32 bounds cannot decide most simplices
    (the prefilter must defer them to binary64)."""
    pts = _lattice(3, 14, jitter=1e-9, seed=5)
    rng = np.random.default_rng(2)
    sid = np.sort(rng.choice(len(pts), size=len(pts) // 16, replace=False)).astype(np.uint32)
    slab = np.minimum((pts[sid, 1] * 3 // 14).astype(np.uint32), 2)
    _check(pts, sid, slab, 3, ctx)


@pytest.mark.parametrize("dim", [2, 3])
def test_degenerate_simplex_raises(dim, ctx):
    """A finite simplex whose vertices have zero exact orientation is the
    reference's DegenerateSimplex (circumsphere, geometry.cpp:279-297): two of
    its vertices are made to coincide. Every policy raises it, without reading
    Simplex::parity for grid / bbox (the check is geometric)."""
    inst = host.make_instance(1 if dim == 2 else 2, n=20_000, k=4)
    lab = oracle.assign_brute(inst.points, inst.sample_ids, inst.sample_labels)
    P = host.attach_partials(inst, lab)
    fin = np.nonzero(P.verts[dim] != 0xFFFFFFFF)[0]
    row = int(fin[len(fin) // 2])
    pts = inst.points.copy()
    pts[P.verts[dim, row]] = pts[P.verts[0, row]]
    for policy in ("grid", "bbox", "exact"):
        with pytest.raises(gpu.DegenerateSimplex):
            gpu.find_border(pts, lab, P, gpu.IntersectionPolicy(policy, 1.0), hull_bfs=False, ctx=ctx)
    # the context stays usable
    g = gpu.find_border(inst.points, lab, P, gpu.IntersectionPolicy("grid", 1.0), hull_bfs=False, ctx=ctx)
    o = oracle.find_border(inst.points, lab, P, "grid")
    assert np.array_equal(g.positive, o["positive"])


def test_grid_policy_does_not_read_parity(ctx):
    """grid / bbox results are independent of Simplex::parity (zeroed here)."""
    inst = host.make_instance(2, n=20_000, k=4)
    lab = oracle.assign_brute(inst.points, inst.sample_ids, inst.sample_labels)
    P = host.attach_partials(inst, lab)
    from paper_1902_07554_b200.host import Partials
    Z = Partials(P.offsets, P.verts, P.nbrs, np.zeros_like(P.parity))
    for policy in ("grid", "bbox"):
        g = gpu.find_border(inst.points, lab, Z, gpu.IntersectionPolicy(policy, 1.0), hull_bfs=True, ctx=ctx)
        o = oracle.find_border(inst.points, lab, P, policy)
        assert np.array_equal(g.positive, o["positive"]), policy
        assert np.array_equal(g.border, o["border"]), policy


def test_exact_policy_partition_without_rows(ctx):
    """Exact policy: a partition holding points but too few for a simplex (2
    points in 3-D: no rows, hence no hull facets) leaves the hull vertex set
    incomplete; the hull rows must then take the leaf-scan descent, and its
    points still count as foreign points for every other partition."""
    inst = host.make_instance(2, n=20_000, k=4)
    lab = oracle.assign_brute(inst.points, inst.sample_ids, inst.sample_labels).copy()
    # two points near the domain's lower corner become partition 4
    far = np.argsort(inst.points.sum(axis=1))[:2]
    lab[far] = 4
    # the DTs of parts 0..3; part 4 (2 points) has none: an empty row range
    tris = [host.triangulate(inst.points, np.nonzero(lab == p)[0].astype(np.uint32), 7) for p in range(4)]
    offs = np.zeros(6, np.uint64)
    offs[1:5] = np.cumsum([t.verts.shape[1] for t in tris])
    offs[5] = offs[4]
    P5 = host.Partials(offs, np.concatenate([t.verts for t in tris], axis=1),
                       np.concatenate([t.nbrs for t in tris], axis=1), np.concatenate([t.parity for t in tris]))
    g = gpu.find_border(inst.points, lab, P5, gpu.IntersectionPolicy("exact", 1.0), hull_bfs=True, ctx=ctx)
    o = oracle.find_border(inst.points, lab, P5, "exact")
    assert np.array_equal(g.positive, o["positive"])
    assert np.array_equal(g.border, o["border"])
    assert np.array_equal(g.positive_vertex_ids, o["vertices_positive"])


def test_bucketing_many_partitions(ctx):
    """k = 3000 > the shared-memory label chunk of the bucketing kernels (1024):
    Partitioning.parts over several label passes, ids ascending per part."""
    rng = np.random.default_rng(11)
    pts = np.ascontiguousarray(rng.random((200_000, 3)))
    sid = np.sort(rng.choice(len(pts), 6000, replace=False)).astype(np.uint32)
    slab = (np.arange(6000) % 3000).astype(np.uint32)
    part = gpu.assign_points(pts, sid, slab, 3000, ctx=ctx)
    ref = oracle.assign_brute(pts, sid, slab)
    assert np.array_equal(part.labels, ref)
    order = np.lexsort((np.arange(len(ref)), ref)).astype(np.uint32)
    counts = np.bincount(ref, minlength=3000)
    assert np.array_equal(part.parts_offsets, np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64))
    assert np.array_equal(part.parts_ids, order)


def test_find_border_many_partitions(ctx):
    """k = 1200: the part offsets no longer fit the kernels' shared memory and
    the bbox policy's per-partition boxes go straight to global memory."""
    inst = host.make_instance(dict(name="manyk", dist="uniform", dim=3, n=60_000, seed=5, frac=0.05, k=1200))
    lab = oracle.assign_kdtree(inst.points, inst.sample_ids, inst.sample_labels)
    P = host.build_partials(inst.points, lab, 1200, 3)
    for policy in ("grid", "bbox", "exact"):
        g = gpu.find_border(inst.points, lab, P, gpu.IntersectionPolicy(policy, 1.0), hull_bfs=True, ctx=ctx)
        o = oracle.find_border(inst.points, lab, P, policy)
        assert np.array_equal(g.positive, o["positive"]), policy
        assert np.array_equal(g.border, o["border"]), policy
        assert np.array_equal(g.positive_vertex_ids, o["vertices_positive"]), policy


def _grid_parts(dim, n, side, seed):
    """Points labelled by a side^dim grid of parts (a few points per part);
    parts with fewer than dim + 1 points get an empty row range."""
    rng = np.random.default_rng(seed)
    pts = np.ascontiguousarray(rng.random((n, dim)))
    cell = np.minimum((pts * side).astype(np.int64), side - 1)
    lab = np.zeros(n, np.int64)
    for d in range(dim):
        lab = lab * side + cell[:, d]
    lab = lab.astype(np.uint32)
    k = side ** dim
    tris = [host.triangulate(pts, np.nonzero(lab == p)[0].astype(np.uint32), 7)
            if np.count_nonzero(lab == p) > dim else None for p in range(k)]
    offs = np.zeros(k + 1, np.uint64)
    offs[1:] = np.cumsum([t.verts.shape[1] if t else 0 for t in tris])
    T = [t for t in tris if t]
    P = host.Partials(offs, np.concatenate([t.verts for t in T], 1), np.concatenate([t.nbrs for t in T], 1),
                      np.concatenate([t.parity for t in T]))
    return pts, lab, P


def test_tiny_parts_mostly_hull_rows(ctx):
    """~3 points per part (k = 4096, 3-D): two thirds of all rows are hull
    (infinite) rows — more than half, the old hull-queue capacity."""
    pts, lab, P = _grid_parts(3, 12_000, 16, 21)
    assert np.count_nonzero(P.verts[3] == 0xFFFFFFFF) > 0.6 * P.S
    for policy in ("grid", "exact"):
        g = gpu.find_border(pts, lab, P, gpu.IntersectionPolicy(policy, 1.0), hull_bfs=True, ctx=ctx)
        o = oracle.find_border(pts, lab, P, policy)
        assert np.array_equal(g.positive, o["positive"]), policy
        assert np.array_equal(g.border, o["border"]), policy
        assert np.array_equal(g.positive_vertex_ids, o["vertices_positive"]), policy


def test_sample_label_out_of_range(ctx):
    """A sample label >= k is rejected (the C++ header's precondition,
    include/sbdt/sample_partition.hpp): up front by the host-buffer entry
    point, and by the bucketing pass's count check on the device path."""
    import torch
    rng = np.random.default_rng(9)
    pts = np.ascontiguousarray(rng.random((5000, 3)))
    sid = np.arange(0, 5000, 50, dtype=np.uint32)
    slab = (np.arange(len(sid)) % 4).astype(np.uint32)
    slab[7] = 4  # k = 4
    with pytest.raises(ValueError):
        gpu.assign_points(pts, sid, slab, 4, ctx=ctx)
    dev = torch.device("cuda", 0)
    d_xyz = torch.from_numpy(pts).to(dev)
    d_sid = torch.from_numpy(sid.view(np.int32)).to(dev)
    d_slab = torch.from_numpy(slab.view(np.int32)).to(dev)
    d_lab = torch.empty(5000, dtype=torch.int32, device=dev)
    d_off = torch.empty(5, dtype=torch.int64, device=dev)
    d_ids = torch.empty(5000, dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    ctx.assign_points_dev(3, d_xyz.data_ptr(), 5000, d_sid.data_ptr(), d_slab.data_ptr(), len(sid), 4,
                          d_lab.data_ptr(), d_off.data_ptr(), d_ids.data_ptr())
    with pytest.raises(ValueError):
        ctx.synchronize()
    ctx.synchronize()  # the status was consumed: the context stays usable
    slab[7] = 3
    part = gpu.assign_points(pts, sid, slab, 4, ctx=ctx)
    assert np.array_equal(part.labels, oracle.assign_brute(pts, sid, slab))


@pytest.mark.parametrize("policy", ["grid", "exact", "bbox"])
def test_recursion_level_grid(policy, ctx):
    """find_border at a recursion level: the level's points
    are a subset (the others labelled UNINDEXED: no cell, no foreign point)
    and the grid is the top level's (global bbox + n_total)."""
    inst = host.make_instance(2, n=60_000, k=8)
    lab = oracle.assign_brute(inst.points, inst.sample_ids, inst.sample_labels)
    P = host.attach_partials(inst, lab)
    L = 5
    SL = int(P.offsets[L])
    lvl_lab = np.where(lab < L, lab, np.uint32(gpu.UNINDEXED)).astype(np.uint32)
    lvl = host.Partials(P.offsets[:L + 1].copy(), np.ascontiguousarray(P.verts[:, :SL]),
                        np.ascontiguousarray(P.nbrs[:, :SL]), P.parity[:SL].copy())
    lo, hi = inst.points.min(axis=0), inst.points.max(axis=0)
    g = gpu.find_border(inst.points, lvl_lab, lvl, gpu.IntersectionPolicy(policy, 1.0), hull_bfs=True, ctx=ctx,
                        grid_bbox=(lo, hi), grid_n_total=inst.n)
    o = oracle.find_border(inst.points, lvl_lab, lvl, policy, grid_bbox=(lo, hi), grid_n_total=inst.n)
    assert np.array_equal(g.positive, o["positive"]) and np.array_equal(g.border, o["border"])
    assert np.array_equal(g.positive_vertex_ids, o["vertices_positive"])
    assert np.array_equal(g.border_vertex_ids, o["vertices_border"])


@pytest.mark.parametrize("dim", [2, 3])
def test_elongated_bbox_grid_capacity(dim, ctx):
    """A bbox far from cubical (a thin needle / strip): c_G (V/n)^(1/D) cells
    along the long axis far exceed the default 4 n capacity; the host entry
    point retries with the capacity the grid needs instead of failing."""
    rng = np.random.default_rng(17 + dim)
    n = 20_000
    pts = rng.random((n, dim))
    pts[:, 1:] *= 1e-6 if dim == 3 else 1e-9
    pts = np.ascontiguousarray(pts)
    lab = np.minimum((pts[:, 0] * 4).astype(np.uint32), 3)
    P = host.build_partials(pts, lab, 4, 7)
    _, _, _, dims = oracle.grid_params(pts, 1.0)
    assert np.prod(dims) > 4 * n  # beyond the default capacity
    for policy in ("grid", "exact"):
        g = gpu.find_border(pts, lab, P, gpu.IntersectionPolicy(policy, 1.0), hull_bfs=True, ctx=ctx)
        o = oracle.find_border(pts, lab, P, policy)
        assert np.array_equal(g.positive, o["positive"]), policy
        assert np.array_equal(g.border, o["border"]), policy
        assert np.array_equal(g.positive_vertex_ids, o["vertices_positive"]), policy


@pytest.mark.parametrize("dim", [2, 3])
def test_enclosed_island_bfs(dim, ctx):
    """Part 1 is an island (the samples within 0.15 of the centre) inside
    part 0: part 0's simplices around the hole are positive but their
    component holds no hull simplex, so the SPEC BFS border (find_border,
    SPEC.md:491) is a strict subset of the full-scan positive set and the
    hull-BFS takes its general path (per-row root marks, not the all-reached
    copy)."""
    inst = host.make_instance(1 if dim == 2 else 2, n=30_000, k=2)
    sp = inst.points[inst.sample_ids]
    sl = (np.linalg.norm(sp - 0.5, axis=1) < 0.15).astype(np.uint32)
    lab = oracle.assign_brute(inst.points, inst.sample_ids, sl)
    P = host.build_partials(inst.points, lab, 2, 7)
    for policy in ("grid", "exact"):
        o = oracle.find_border(inst.points, lab, P, policy)
        assert o["border"].sum() < o["positive"].sum()
        for _ in range(4):  # the union-find runs with concurrent hooks: repeat
            g = gpu.find_border(inst.points, lab, P, gpu.IntersectionPolicy(policy, 1.0), hull_bfs=True, ctx=ctx)
            assert np.array_equal(g.positive, o["positive"])
            assert np.array_equal(g.border, o["border"])
            assert np.array_equal(g.positive_vertex_ids, o["vertices_positive"])
            assert np.array_equal(g.border_vertex_ids, o["vertices_border"])
