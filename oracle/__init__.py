"""TEST INFRASTRUCTURE — the CPU oracle (checker) for the hot path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this package. It is never on the product
path: the product (paper_1902_07554_b200, libsbdt_gpu.so) does not load it.

liboracle.so  : restatement of SPEC.md assign_points (kd-tree + brute force),
                GridIndex / intersects_* and find_border (oracle/path.hpp) on
                restated primitives (oracle/prims.hpp); merge +
                update_neighbors (oracle/merge.hpp).
_ref/libsbdt_ref.so : the same path templates instantiated on the reference's
                own geometry.cpp / triangulation.cpp / sequential_dt.cpp
                (compiled by path in this container; pins the restatement).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_oracle = None
_ref = None

POLICY = {"bbox": 0, "grid": 1, "exact": 2}


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def lib():
    global _oracle
    if _oracle is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError("oracle/liboracle.so missing: run `make -C oracle`")
        L = C.CDLL(path)
        u64, u32p, dp, i8p, u8p = C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_double), C.POINTER(C.c_int8), C.POINTER(C.c_uint8)
        L.oracle_assign_brute.argtypes = [C.c_int, dp, u64, u32p, u64, u32p, u32p, C.c_int]
        L.oracle_assign_kdtree.argtypes = [C.c_int, dp, u64, u32p, u64, u32p, u32p, C.c_int]
        L.oracle_assign_kdtree_range.argtypes = [C.c_int, dp, u64, u64, u32p, u64, u32p, u32p, C.c_int]
        L.oracle_grid_params.argtypes = [C.c_int, dp, u64, C.c_double, dp, dp, dp, C.POINTER(C.c_int64)]
        L.oracle_find_border.argtypes = [C.c_int, dp, u64, u32p, C.c_uint32, C.POINTER(C.c_uint64), u32p, u32p, i8p,
                                         C.c_int, C.c_double, C.c_int, C.c_uint32, C.c_uint32, u8p, u8p, u32p,
                                         C.POINTER(C.c_uint64), u32p, C.POINTER(C.c_uint64), dp, dp, dp, u64,
                                         C.c_char_p, C.c_int]
        L.oracle_time_border.argtypes = [C.c_int, dp, u64, u32p, C.c_uint32, C.POINTER(C.c_uint64), u32p, u32p, i8p,
                                         C.c_int, C.c_double, C.c_int, C.c_uint32, C.c_uint32, C.c_int, dp, dp,
                                         C.POINTER(C.c_uint64)]
        L.oracle_merge.restype = C.c_void_p
        L.oracle_merge.argtypes = [C.c_int, C.c_uint32, C.POINTER(C.c_uint64), u32p, u32p, i8p, u8p, u32p, u32p, i8p,
                                   u64, u32p, C.c_int, C.c_char_p, C.c_int]
        L.oracle_merge_rows.restype = u64
        L.oracle_merge_rows.argtypes = [C.c_void_p]
        L.oracle_merge_export.argtypes = [C.c_void_p, u32p, u32p, i8p, C.POINTER(C.c_uint64)]
        L.oracle_merge_free.argtypes = [C.c_void_p]
        L.oracle_orient.argtypes = [C.c_int, dp]
        L.oracle_in_sphere.argtypes = [C.c_int, dp, dp]
        L.oracle_circumsphere.argtypes = [C.c_int, dp, dp]
        L.oracle_orient_batch.argtypes = [C.c_int, dp, u64, C.POINTER(C.c_int8)]
        L.oracle_in_sphere_batch.argtypes = [C.c_int, dp, u64, C.POINTER(C.c_int8)]
        L.oracle_box_sphere.argtypes = [C.c_int, dp, dp, dp, C.c_double]
        L.oracle_halfspace_box.argtypes = [C.c_int, dp, dp, dp, dp]
        _oracle = L
    return _oracle


def ref_lib():
    """The reference's own compiled primitives (None if oracle/_ref was not built)."""
    global _ref
    if _ref is None:
        path = os.path.join(_HERE, "_ref", "libsbdt_ref.so")
        if not os.path.exists(path):
            return None
        L = C.CDLL(path)
        u64, u32p, dp, i8p, u8p = C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_double), C.POINTER(C.c_int8), C.POINTER(C.c_uint8)
        L.ref_orient.argtypes = [C.c_int, dp]
        L.ref_in_sphere.argtypes = [C.c_int, dp, dp]
        L.ref_circumsphere.argtypes = [C.c_int, dp, dp]
        L.ref_orient_batch.argtypes = [C.c_int, dp, u64, C.POINTER(C.c_int8)]
        L.ref_in_sphere_batch.argtypes = [C.c_int, dp, u64, C.POINTER(C.c_int8)]
        L.ref_inflate.restype = C.c_double
        L.ref_inflate.argtypes = [C.c_double]
        L.ref_box_sphere.argtypes = [C.c_int, dp, dp, dp, C.c_double]
        L.ref_halfspace_box.argtypes = [C.c_int, dp, dp, dp, dp]
        L.ref_triangulate.restype = C.c_void_p
        L.ref_triangulate.argtypes = [C.c_int, dp, u64, u32p, u64, u64]
        L.ref_tri_count.restype = u64
        L.ref_tri_count.argtypes = [C.c_void_p]
        L.ref_tri_export.argtypes = [C.c_void_p, u32p, u32p, i8p]
        L.ref_tri_free.argtypes = [C.c_void_p]
        L.ref_assign_brute.argtypes = [C.c_int, dp, u64, u32p, u64, u32p, u32p]
        L.ref_find_border.argtypes = [C.c_int, dp, u64, u32p, C.c_uint32, C.POINTER(C.c_uint64), u32p, u32p, i8p,
                                      C.c_int, C.c_double, u8p, u8p, u32p, C.POINTER(C.c_uint64), u32p,
                                      C.POINTER(C.c_uint64)]
        L.ref_time_step.argtypes = [C.c_int, dp, u64, u32p, u64, u32p, u64, u32p, C.c_uint32, C.POINTER(C.c_uint64),
                                    u32p, u32p, i8p, C.c_int, C.c_double, C.c_uint, C.c_uint32, C.c_uint32, u32p, u8p,
                                    dp, C.POINTER(C.c_uint64)]
        _ref = L
    return _ref


# ---------------------------------------------------------------------------
def assign_brute(points, sample_ids, sample_labels, threads=8):
    pts = np.ascontiguousarray(points, np.float64)
    sid = np.ascontiguousarray(sample_ids, np.uint32)
    slab = np.ascontiguousarray(sample_labels, np.uint32)
    out = np.empty(len(pts), np.uint32)
    lib().oracle_assign_brute(pts.shape[1], _p(pts, C.c_double), len(pts), _p(sid, C.c_uint32), len(sid),
                              _p(slab, C.c_uint32), _p(out, C.c_uint32), threads)
    return out


def assign_kdtree(points, sample_ids, sample_labels, threads=8):
    pts = np.ascontiguousarray(points, np.float64)
    sid = np.ascontiguousarray(sample_ids, np.uint32)
    slab = np.ascontiguousarray(sample_labels, np.uint32)
    out = np.empty(len(pts), np.uint32)
    lib().oracle_assign_kdtree(pts.shape[1], _p(pts, C.c_double), len(pts), _p(sid, C.c_uint32), len(sid),
                               _p(slab, C.c_uint32), _p(out, C.c_uint32), threads)
    return out


def grid_params(points, c_G=1.0):
    pts = np.ascontiguousarray(points, np.float64)
    dim = pts.shape[1]
    lo, hi, edge, dims = np.empty(dim), np.empty(dim), np.empty(1), np.empty(dim, np.int64)
    lib().oracle_grid_params(dim, _p(pts, C.c_double), len(pts), c_G, _p(lo, C.c_double), _p(hi, C.c_double),
                             _p(edge, C.c_double), _p(dims, C.c_int64))
    return lo, hi, float(edge[0]), dims


def find_border(points, labels, partials, policy="grid", c_G=1.0, threads=8, parts=None, spheres=False,
                grid_bbox=None, grid_n_total=0):
    """Returns dict(positive, border, vertices_positive, vertices_border, times[, spheres]);
    times = (index build s, find_border s) measured inside the library."""
    pts = np.ascontiguousarray(points, np.float64)
    lab = np.ascontiguousarray(labels, np.uint32)
    dim = pts.shape[1]
    S = partials.S
    k = partials.k
    p0, p1 = (0, 0) if parts is None else parts
    pos = np.empty(S, np.uint8)
    bor = np.empty(S, np.uint8)
    vpos = np.empty(len(pts), np.uint32)
    vbfs = np.empty(len(pts), np.uint32)
    npos, nbfs = C.c_uint64(0), C.c_uint64(0)
    sph = np.empty((S, dim + 1), np.float64) if spheres else None
    err = C.create_string_buffer(256)
    times = np.zeros(2)
    gbb = None if grid_bbox is None else np.ascontiguousarray(np.concatenate([np.asarray(grid_bbox[0], np.float64),
                                                                              np.asarray(grid_bbox[1], np.float64)]))
    rc = lib().oracle_find_border(dim, _p(pts, C.c_double), len(pts), _p(lab, C.c_uint32), k,
                                  _p(partials.offsets, C.c_uint64), _p(partials.verts, C.c_uint32),
                                  _p(partials.nbrs, C.c_uint32), _p(partials.parity, C.c_int8), POLICY[policy], c_G,
                                  threads, p0, p1, _p(pos, C.c_uint8), _p(bor, C.c_uint8), _p(vpos, C.c_uint32),
                                  C.byref(npos), _p(vbfs, C.c_uint32), C.byref(nbfs),
                                  _p(sph, C.c_double) if spheres else None, _p(times, C.c_double),
                                  _p(gbb, C.c_double) if gbb is not None else None, int(grid_n_total), err, 256)
    if rc != 0:
        raise RuntimeError("oracle_find_border: " + err.value.decode())
    out = dict(positive=pos, border=bor, vertices_positive=vpos[:npos.value].copy(),
               vertices_border=vbfs[:nbfs.value].copy(), times=(float(times[0]), float(times[1])))
    if spheres:
        out["spheres"] = sph
    return out


def time_border(points, labels, partials, policy="grid", c_G=1.0, threads=8, parts=(0, 0), reps=1):
    pts = np.ascontiguousarray(points, np.float64)
    lab = np.ascontiguousarray(labels, np.uint32)
    tb, tr = C.c_double(0), C.c_double(0)
    nv = C.c_uint64(0)
    lib().oracle_time_border(pts.shape[1], _p(pts, C.c_double), len(pts), _p(lab, C.c_uint32), partials.k,
                             _p(partials.offsets, C.c_uint64), _p(partials.verts, C.c_uint32),
                             _p(partials.nbrs, C.c_uint32), _p(partials.parity, C.c_int8), POLICY[policy], c_G,
                             threads, parts[0], parts[1] or partials.k, reps, C.byref(tb), C.byref(tr), C.byref(nv))
    return tb.value, tr.value, nv.value


def merge(partials, border, tb, labels, hull=True):
    """SPEC.md:497-514 merge + update_neighbors (oracle/merge.hpp). `border`:
    per partial row, nonzero = border simplex; `tb`: the border triangulation
    (verts/nbrs (D+1, S_B), parity). Returns (verts, nbrs, parity, offsets)."""
    dim = partials.verts.shape[0] - 1
    bor = np.ascontiguousarray(border, np.uint8)
    lab = np.ascontiguousarray(labels, np.uint32)
    tv = np.ascontiguousarray(tb.verts, np.uint32)
    tn = np.ascontiguousarray(tb.nbrs, np.uint32)
    tp = np.ascontiguousarray(tb.parity, np.int8)
    err = C.create_string_buffer(256)
    h = lib().oracle_merge(dim, partials.k, _p(partials.offsets, C.c_uint64), _p(partials.verts, C.c_uint32),
                           _p(partials.nbrs, C.c_uint32), _p(partials.parity, C.c_int8), _p(bor, C.c_uint8),
                           _p(tv, C.c_uint32), _p(tn, C.c_uint32), _p(tp, C.c_int8), tv.shape[1],
                           _p(lab, C.c_uint32), int(hull), err, 256)
    if not h:
        raise RuntimeError("oracle_merge: " + err.value.decode())
    try:
        R = lib().oracle_merge_rows(h)
        v = np.empty((dim + 1, R), np.uint32)
        nb = np.empty((dim + 1, R), np.uint32)
        par = np.empty(R, np.int8)
        off = np.empty(partials.k + 3, np.uint64)
        lib().oracle_merge_export(h, _p(v, C.c_uint32), _p(nb, C.c_uint32), _p(par, C.c_int8), _p(off, C.c_uint64))
    finally:
        lib().oracle_merge_free(h)
    return v, nb, par, off


def ref_time_step(points, sample_ids, sample_labels, labels, partials, policy="grid", c_G=1.0, threads=1,
                  n_assign=None, parts=(0, 0)):
    """One CPU step of the path on the reference's own compiled primitives and
    its TaskPool(threads) (oracle/_ref; None if it was not built): kd-tree
    assign_points over points [0, n_assign), then find_border over parts
    [p0, p1) with `labels`. Returns dict(labels, positive, times=(assign,
    index build, border) seconds, border_vertices)."""
    L = ref_lib()
    if L is None:
        return None
    pts = np.ascontiguousarray(points, np.float64)
    sid = np.ascontiguousarray(sample_ids, np.uint32)
    slab = np.ascontiguousarray(sample_labels, np.uint32)
    lab = np.ascontiguousarray(labels, np.uint32)
    n = len(pts)
    na = n if n_assign is None else int(n_assign)
    out_lab = np.empty(max(na, 1), np.uint32)
    pos = np.zeros(partials.S, np.uint8)
    times = np.zeros(3)
    nvb = C.c_uint64(0)
    rc = L.ref_time_step(pts.shape[1], _p(pts, C.c_double), n, _p(sid, C.c_uint32), len(sid), _p(slab, C.c_uint32),
                         na, _p(lab, C.c_uint32), partials.k, _p(partials.offsets, C.c_uint64),
                         _p(partials.verts, C.c_uint32), _p(partials.nbrs, C.c_uint32), _p(partials.parity, C.c_int8),
                         POLICY[policy], c_G, threads, parts[0], parts[1], _p(out_lab, C.c_uint32),
                         _p(pos, C.c_uint8), _p(times, C.c_double), C.byref(nvb))
    if rc != 0:
        raise RuntimeError("ref_time_step failed")
    return dict(labels=out_lab[:na], positive=pos, times=tuple(float(t) for t in times),
                border_vertices=int(nvb.value))


def cpu_model() -> str:
    """Host CPU model string (/proc/cpuinfo) for the baseline records."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def predicates_batch(op, pts, use_ref=True):
    """orient / in_sphere signs of the cases in `pts` (layout of
    gpu.Context.predicates), by the reference's compiled geometry.cpp when
    oracle/_ref exists (use_ref), else by the restatement. Returns (signs, which)."""
    pts = np.ascontiguousarray(pts, np.float64)
    count, _, dim = pts.shape
    out = np.empty(count, np.int8)
    L = ref_lib() if use_ref else None
    if L is not None:
        fn, which = (L.ref_orient_batch if op == "orient" else L.ref_in_sphere_batch), "reference"
    else:
        fn, which = (lib().oracle_orient_batch if op == "orient" else lib().oracle_in_sphere_batch), "oracle"
    fn(dim, _p(pts, C.c_double), count, _p(out, C.c_int8))
    return out, which
