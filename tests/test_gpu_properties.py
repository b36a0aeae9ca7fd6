"""GPU tests beyond the small parity grid: the prefilter path (no sphere
export), larger instances checked against the oracle on a bounded subset
(first points / first parts), size-independent properties (policy chain,
BFS subset, determinism, Partitioning consistency) and error behaviour."""
import numpy as np
import pytest

import oracle
from paper_1902_07554_b200 import gpu, host

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,n,k", [(1, 200_000, 16), (2, 300_000, 16), (3, 300_000, 16), (4, 400_000, 32),
                                     (5, 600_000, 32)])
def test_prefilter_path_bit_exact(cfg, n, k, ctx):
    inst = host.make_instance(cfg, n=n, k=k)
    lab = gpu.assign_points(inst.points, inst.sample_ids, inst.sample_labels, k, ctx=ctx).labels
    ref = oracle.assign_kdtree(inst.points, inst.sample_ids, inst.sample_labels)
    assert np.array_equal(lab, ref)
    part = host.attach_partials(inst, lab)
    g = gpu.find_border(inst.points, lab, part, gpu.IntersectionPolicy("grid", 1.0), hull_bfs=True, ctx=ctx)
    o = oracle.find_border(inst.points, lab, part, "grid")
    assert np.array_equal(g.positive, o["positive"])
    assert np.array_equal(g.border, o["border"])
    assert np.array_equal(g.positive_vertex_ids, o["vertices_positive"])
    assert np.array_equal(g.border_vertex_ids, o["vertices_border"])


def test_large_instance_subset_parity(ctx):
    """Config 2 at 2M points (k=64): labels of the first 300k points and the
    flags of the first 6 parts against the oracle (bounded CPU work)."""
    inst = host.make_instance(2, n=2_000_000, k=64)
    part_ = gpu.assign_points(inst.points, inst.sample_ids, inst.sample_labels, 64, ctx=ctx)
    sub = slice(0, 300_000)
    # oracle on a prefix of the points (the kd-tree still spans the whole sample)
    full_ref = np.empty(300_000, np.uint32)
    import ctypes as C
    pts = np.ascontiguousarray(inst.points)
    oracle.lib().oracle_assign_kdtree_range(3, oracle._p(pts, C.c_double), 0, 300_000,
                                            oracle._p(inst.sample_ids, C.c_uint32), len(inst.sample_ids),
                                            oracle._p(inst.sample_labels, C.c_uint32), oracle._p(full_ref, C.c_uint32),
                                            8)
    assert np.array_equal(part_.labels[sub], full_ref)
    lab = part_.labels
    part = host.attach_partials(inst, lab)
    g = gpu.find_border(inst.points, lab, part, gpu.IntersectionPolicy("grid", 1.0), hull_bfs=True, ctx=ctx)
    o = oracle.find_border(inst.points, lab, part, "grid", parts=(0, 6))
    hi = int(part.offsets[6])
    assert np.array_equal(g.positive[:hi], o["positive"][:hi])
    assert np.array_equal(g.border[:hi], o["border"][:hi])


def test_policy_chain_and_subsets(ctx):
    inst = host.make_instance(4, n=300_000, k=16)
    lab = gpu.assign_points(inst.points, inst.sample_ids, inst.sample_labels, 16, ctx=ctx).labels
    part = host.attach_partials(inst, lab)
    grid = gpu.find_border(inst.points, lab, part, gpu.IntersectionPolicy("grid"), ctx=ctx)
    bbox = gpu.find_border(inst.points, lab, part, gpu.IntersectionPolicy("bbox"), ctx=ctx)
    exact = gpu.find_border(inst.points, lab, part, gpu.IntersectionPolicy("exact"), ctx=ctx)
    assert set(grid.border_vertex_ids.tolist()) <= set(bbox.border_vertex_ids.tolist())
    assert np.all(grid.positive <= bbox.positive)
    # exact <= grid <= bbox
    assert np.all(exact.positive <= grid.positive)
    assert set(exact.border_vertex_ids.tolist()) <= set(grid.border_vertex_ids.tolist())
    o = oracle.find_border(inst.points, lab, part, "exact")
    assert np.array_equal(exact.positive, o["positive"]) and np.array_equal(exact.border, o["border"])
    assert np.all(grid.border <= grid.positive)  # BFS subset of the full scan
    assert set(grid.border_vertex_ids.tolist()) <= set(grid.positive_vertex_ids.tolist())
    again = gpu.find_border(inst.points, lab, part, gpu.IntersectionPolicy("grid"), ctx=ctx)
    assert np.array_equal(again.positive, grid.positive) and np.array_equal(again.border_vertex_ids,
                                                                             grid.border_vertex_ids)


def test_partitioning_consistency_and_determinism(ctx):
    inst = host.make_instance(5, n=500_000, k=64)
    a = gpu.assign_points(inst.points, inst.sample_ids, inst.sample_labels, 64, ctx=ctx)
    b = gpu.assign_points(inst.points, inst.sample_ids, inst.sample_labels, 64, ctx=ctx)
    assert np.array_equal(a.labels, b.labels) and np.array_equal(a.parts_ids, b.parts_ids)
    assert a.parts_offsets[-1] == inst.n
    for p in range(64):
        ids = a.part(p)
        assert np.all(np.diff(ids.astype(np.int64)) > 0)
        assert np.all(a.labels[ids] == p)


def test_sample_points_label_themselves(ctx):
    inst = host.make_instance(1, n=50_000, k=8)
    lab = gpu.assign_points(inst.points, inst.sample_ids, inst.sample_labels, 8, ctx=ctx).labels
    assert np.array_equal(lab[inst.sample_ids], inst.sample_labels)


def test_invalid_arguments_raise(ctx):
    pts = np.random.default_rng(0).random((100, 2))
    with pytest.raises(ValueError):
        gpu.assign_points(pts, np.array([], np.uint32), np.array([], np.uint32), 4, ctx=ctx)
    with pytest.raises(ValueError):
        gpu.assign_points(np.random.default_rng(0).random((100, 4)), np.array([0], np.uint32),
                          np.array([0], np.uint32), 1, ctx=ctx)


def test_k1_no_border(ctx):
    inst = host.make_instance(1, n=20_000, k=1)
    lab = np.zeros(inst.n, np.uint32)
    part = host.attach_partials(inst, lab)
    g = gpu.find_border(inst.points, lab, part, ctx=ctx)
    assert g.positive.sum() == 0 and len(g.border_vertex_ids) == 0


def test_pinned_output_buffers_match(ctx):
    """out= buffers (page-locked) give the same results as fresh arrays, with
    and without the BFS (the no-BFS host path uploads only the last neighbour row)."""
    inst = host.make_instance(2, n=100_000, k=16)
    a = gpu.assign_points(inst.points, inst.sample_ids, inst.sample_labels, 16, ctx=ctx)
    out_a = gpu.Partitioning(gpu.pinned_empty(inst.n, np.uint32), gpu.pinned_empty(17, np.uint64),
                             gpu.pinned_empty(inst.n, np.uint32), inst.sample_ids, inst.sample_labels,
                             gpu.pinned_empty(6, np.float64))
    b = gpu.assign_points(inst.points, inst.sample_ids, inst.sample_labels, 16, ctx=ctx, out=out_a)
    assert b.labels is out_a.labels
    assert np.array_equal(a.labels, b.labels) and np.array_equal(a.parts_ids, b.parts_ids)
    part = host.attach_partials(inst, a.labels)
    ref = gpu.find_border(inst.points, a.labels, part, gpu.IntersectionPolicy("grid"), ctx=ctx)
    S = part.S
    out_b = gpu.BorderSet(gpu.pinned_empty(S, np.uint8), gpu.pinned_empty(S, np.uint8),
                          gpu.pinned_empty(inst.n, np.uint32), gpu.pinned_empty(inst.n, np.uint32))
    got = gpu.find_border(inst.points, a.labels, part, gpu.IntersectionPolicy("grid"), ctx=ctx, out=out_b)
    assert np.array_equal(got.positive, ref.positive) and np.array_equal(got.border, ref.border)
    assert np.array_equal(got.border_vertex_ids, ref.border_vertex_ids)
    assert np.array_equal(got.positive_vertex_ids, ref.positive_vertex_ids)
    nob = gpu.find_border(inst.points, a.labels, part, gpu.IntersectionPolicy("grid"), hull_bfs=False, ctx=ctx)
    assert np.array_equal(nob.positive, ref.positive)
    assert np.array_equal(nob.positive_vertex_ids, ref.positive_vertex_ids)
    with pytest.raises(ValueError):
        gpu.find_border(inst.points, a.labels, part, ctx=ctx,
                        out=gpu.BorderSet(np.empty(S + 1, np.uint8), None, None, np.empty(inst.n, np.uint32)))


def test_host_path_equals_device_path(ctx):
    """The host-buffer entry points (chunked uploads overlapping the kernels,
    queue cursors resumed across chunk launches) give the same results as the
    device-pointer entry points on one instance."""
    import torch
    inst = host.make_instance(2, n=300_000, k=16)
    part = gpu.assign_points(inst.points, inst.sample_ids, inst.sample_labels, 16, ctx=ctx)
    pt = host.attach_partials(inst, part.labels)
    hb = gpu.find_border(inst.points, part.labels, pt, gpu.IntersectionPolicy("grid"), hull_bfs=False, ctx=ctx)
    dev = torch.device("cuda", 0)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).to(dev)  # noqa: E731
    d_xyz = torch.from_numpy(np.ascontiguousarray(inst.points)).to(dev)
    d_sid, d_slab = t(inst.sample_ids, np.int32), t(inst.sample_labels, np.int32)
    d_lab = torch.empty(inst.n, dtype=torch.int32, device=dev)
    d_bbox = torch.empty(6, dtype=torch.int64, device=dev)
    dctx = gpu.Context(0)  # device-pointer path on torch's stream
    dctx.set_stream(torch.cuda.current_stream().cuda_stream)
    dctx.assign_points_dev(inst.dim, d_xyz.data_ptr(), inst.n, d_sid.data_ptr(), d_slab.data_ptr(),
                          len(inst.sample_ids), 16, d_lab.data_ptr(), None, None, d_bbox.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(d_lab.cpu().numpy().view(np.uint32), part.labels)
    S = pt.S
    a = gpu.BorderArgs()
    keep = [d_xyz, d_lab, d_bbox]
    d_off, d_v, d_n, d_p = t(pt.offsets, np.int64), t(pt.verts, np.int32), t(pt.nbrs, np.int32), t(pt.parity, np.int8)
    d_pos = torch.empty(S, dtype=torch.uint8, device=dev)
    d_vf = torch.empty(inst.n + 64, dtype=torch.uint8, device=dev)
    d_vids = torch.empty(inst.n, dtype=torch.int32, device=dev)
    d_cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    keep += [d_off, d_v, d_n, d_p, d_pos, d_vf, d_vids, d_cnt]
    a.dim, a.d_xyz, a.n, a.d_labels, a.k = inst.dim, d_xyz.data_ptr(), inst.n, d_lab.data_ptr(), 16
    a.d_offsets, a.d_verts, a.d_nbrs, a.d_parity, a.S = d_off.data_ptr(), d_v.data_ptr(), d_n.data_ptr(), \
        d_p.data_ptr(), S
    a.policy, a.c_G, a.flags = gpu.POLICY["grid"], 1.0, 0
    a.d_bbox_ordered = d_bbox.data_ptr()
    a.d_positive, a.d_vertex_flags, a.d_vertex_ids, a.d_vertex_count = d_pos.data_ptr(), d_vf.data_ptr(), \
        d_vids.data_ptr(), d_cnt.data_ptr()
    dctx.find_border_dev(a)
    torch.cuda.synchronize()
    dctx.synchronize()
    assert np.array_equal(d_pos.cpu().numpy(), hb.positive)
    nv = int(d_cnt.item())
    assert np.array_equal(d_vids[:nv].cpu().numpy().view(np.uint32), hb.positive_vertex_ids)
    dctx.close()


def test_resident_points_flag(ctx):
    """SBDT_BORDER_RESIDENT_POINTS: find_border reuses the device copies of the
    last assign_points call's points and labels; same results, and a call with
    other buffers is rejected."""
    inst = host.make_instance(1, n=80_000, k=8)
    part = gpu.assign_points(inst.points, inst.sample_ids, inst.sample_labels, 8, ctx=ctx)
    pt = host.attach_partials(inst, part.labels)
    res = gpu.find_border(inst.points, part.labels, pt, gpu.IntersectionPolicy("grid"), ctx=ctx, resident=True)
    ref = gpu.find_border(inst.points, part.labels, pt, gpu.IntersectionPolicy("grid"), ctx=ctx)
    assert np.array_equal(res.positive, ref.positive) and np.array_equal(res.border, ref.border)
    assert np.array_equal(res.positive_vertex_ids, ref.positive_vertex_ids)
    with pytest.raises(ValueError):
        gpu.find_border(inst.points.copy(), part.labels, pt, ctx=ctx, resident=True)


def test_zero_copy_hull_neighbours(ctx):
    """No-BFS host call with page-locked partials: the hull rows' neighbours
    are read in place from host memory (zero-copy); same results as the
    pageable (uploaded) path."""
    inst = host.make_instance(2, n=120_000, k=16)
    part = gpu.assign_points(inst.points, inst.sample_ids, inst.sample_labels, 16, ctx=ctx)
    pt = host.attach_partials(inst, part.labels)

    def pinned(a):
        v = gpu.pinned_empty(a.shape, a.dtype)
        v[...] = a
        return v

    pp = host.Partials(pinned(pt.offsets), pinned(pt.verts), pinned(pt.nbrs), pinned(pt.parity))
    zc = gpu.find_border(inst.points, part.labels, pp, gpu.IntersectionPolicy("grid"), hull_bfs=False, ctx=ctx)
    ref = gpu.find_border(inst.points, part.labels, pt, gpu.IntersectionPolicy("grid"), hull_bfs=False, ctx=ctx)
    assert np.array_equal(zc.positive, ref.positive)
    assert np.array_equal(zc.positive_vertex_ids, ref.positive_vertex_ids)
    o = oracle.find_border(inst.points, part.labels, pt, "grid")
    assert np.array_equal(zc.positive, o["positive"])


def _permuted(part, rng):
    """The same partial DTs with each part's rows in a random order
    (neighbour links are part-local row ids: remapped with the permutation)."""
    v, nb, par = part.verts.copy(), part.nbrs.copy(), part.parity.copy()
    for p in range(part.k):
        a, b = int(part.offsets[p]), int(part.offsets[p + 1])
        perm = rng.permutation(b - a)          # new row i holds old row perm[i]
        inv = np.empty_like(perm)
        inv[perm] = np.arange(b - a)
        v[:, a:b] = part.verts[:, a:b][:, perm]
        par[a:b] = part.parity[a:b][perm]
        old_nb = part.nbrs[:, a:b][:, perm]
        nb[:, a:b] = inv[old_nb].astype(np.uint32)
    return host.Partials(part.offsets.copy(), v, nb, par), None


@pytest.mark.parametrize("cfg,n,k", [(2, 200_000, 8), (5, 300_000, 16)])
@pytest.mark.parametrize("order", ["slot", "shuffled"])
def test_find_border_row_order_independent(cfg, n, k, order, ctx, monkeypatch):
    """The host builder emits rows along a Morton curve (a layout decision for
    the device kernels' gathers); find_border must give the same answer for
    any row order: the builder's slot order and a random order per part, each
    against the oracle on the same rows (positive and BFS flags, vertex sets)."""
    inst = host.make_instance(cfg, n=n, k=k)
    lab = oracle.assign_kdtree(inst.points, inst.sample_ids, inst.sample_labels)
    if order == "slot":
        monkeypatch.setenv("SBDT_HOST_ROW_ORDER", "slot")
        part = host.attach_partials(inst, lab)
    else:
        monkeypatch.delenv("SBDT_HOST_ROW_ORDER", raising=False)
        part, _ = _permuted(host.attach_partials(inst, lab), np.random.default_rng(5))
    for policy in ("grid", "exact"):
        g = gpu.find_border(inst.points, lab, part, gpu.IntersectionPolicy(policy, 1.0), hull_bfs=True, ctx=ctx)
        o = oracle.find_border(inst.points, lab, part, policy)
        assert np.array_equal(g.positive, o["positive"])
        assert np.array_equal(g.border, o["border"])
        assert np.array_equal(g.positive_vertex_ids, o["vertices_positive"])
        assert np.array_equal(g.border_vertex_ids, o["vertices_border"])


@pytest.mark.parametrize("seed", [101, 202])
@pytest.mark.parametrize("cfg,n,k", [(1, 300_000, 16), (2, 400_000, 16), (3, 400_000, 16), (4, 500_000, 32),
                                     (5, 600_000, 32)])
def test_other_seeds_bit_exact(cfg, n, k, seed, ctx):
    """The BASELINE configs' distributions under other seeds than the configs'
    own (labels; positive and BFS flags and both vertex sets, grid + exact)."""
    inst = host.make_instance(cfg, n=n, k=k, seed=seed)
    lab = gpu.assign_points(inst.points, inst.sample_ids, inst.sample_labels, k, ctx=ctx).labels
    assert np.array_equal(lab, oracle.assign_kdtree(inst.points, inst.sample_ids, inst.sample_labels))
    part = host.attach_partials(inst, lab)
    for policy in ("grid", "exact"):
        g = gpu.find_border(inst.points, lab, part, gpu.IntersectionPolicy(policy, 1.0), hull_bfs=True, ctx=ctx)
        o = oracle.find_border(inst.points, lab, part, policy)
        assert np.array_equal(g.positive, o["positive"])
        assert np.array_equal(g.border, o["border"])
        assert np.array_equal(g.positive_vertex_ids, o["vertices_positive"])
        assert np.array_equal(g.border_vertex_ids, o["vertices_border"])
