"""Python mirror of the reference's divide-step interface over the C ABI
(include/sbdt_gpu.h -> libsbdt_gpu.so, sm_100a kernels).

Names and argument meaning follow SPEC.md's operations:
  assign_points(P, sample_ids, sample_labels, k) -> Partitioning
  find_border(P, labels, partials, policy)        -> BorderSet
  IntersectionPolicy(kind, c_G)
  merge(partials, border, T_B, labels)            -> Triangulation  SPEC.md:497-514 (+ update_neighbors)
Errors map like the reference's exceptions (common.hpp:22-65). There is no
CPU fallback: a missing library or device raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None

SBDT_OK, SBDT_ERR_INVALID, SBDT_ERR_DEGENERATE, SBDT_ERR_CUDA, SBDT_ERR_OOM, SBDT_ERR_RANGE, SBDT_ERR_MERGE = range(7)
MERGE_HULL = 1
UNINDEXED = 0xFFFFFFFF  # label of a point outside this recursion level's indices (SBDT_UNINDEXED)
POLICY = {"bbox": 0, "grid": 1, "exact": 2}
RESIDENT_POINTS = 2
HULL_BFS = 1


class DegenerateSimplex(RuntimeError):
    """sbdt::DegenerateSimplex (common.hpp:22-25)."""


class SbdtGpuError(RuntimeError):
    pass


class InconsistentMerge(SbdtGpuError):
    """dc-engine InconsistentMerge / DanglingFacet."""


class BorderArgs(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("d_xyz", C.c_void_p), ("n", C.c_uint64), ("d_labels", C.c_void_p), ("k", C.c_uint32),
        ("d_offsets", C.c_void_p), ("d_verts", C.c_void_p), ("d_nbrs", C.c_void_p), ("d_parity", C.c_void_p),
        ("S", C.c_uint64), ("policy", C.c_int), ("c_G", C.c_double), ("flags", C.c_uint32),
        ("d_bbox_ordered", C.c_void_p), ("d_positive", C.c_void_p), ("d_border", C.c_void_p),
        ("d_vertex_flags", C.c_void_p), ("d_vertex_ids", C.c_void_p), ("d_vertex_count", C.c_void_p),
        ("d_bfs_vertex_flags", C.c_void_p), ("d_bfs_vertex_ids", C.c_void_p), ("d_bfs_vertex_count", C.c_void_p),
        ("d_spheres", C.c_void_p), ("grid_bbox", C.POINTER(C.c_double)), ("grid_n_total", C.c_uint64),
        ("grid_max_cells", C.c_uint64),
    ]


class MergeArgs(C.Structure):
    """sbdt_merge_args (include/sbdt_gpu.h)."""
    _fields_ = [
        ("dim", C.c_int), ("k", C.c_uint32), ("d_labels", C.c_void_p), ("n", C.c_uint64), ("d_offsets", C.c_void_p),
        ("d_verts", C.c_void_p), ("d_nbrs", C.c_void_p), ("d_parity", C.c_void_p), ("S", C.c_uint64),
        ("d_border", C.c_void_p), ("d_tb_verts", C.c_void_p), ("d_tb_nbrs", C.c_void_p),
        ("d_tb_parity", C.c_void_p), ("S_B", C.c_uint64), ("flags", C.c_uint32),
    ]


EXPORTS = [
    "sbdt_gpu_host_alloc", "sbdt_gpu_host_free", "sbdt_gpu_create", "sbdt_gpu_destroy", "sbdt_gpu_last_error", "sbdt_gpu_set_stream", "sbdt_gpu_synchronize",
    "sbdt_gpu_launch_count", "sbdt_gpu_check_status", "sbdt_gpu_assign_points", "sbdt_gpu_assign_points_dev",
    "sbdt_gpu_find_border", "sbdt_gpu_find_border_dev", "sbdt_gpu_merge", "sbdt_gpu_merge_dev",
    "sbdt_gpu_set_timing", "sbdt_gpu_stage_times", "sbdt_gpu_assign_table_stats", "sbdt_gpu_border_stats",
    "sbdt_gpu_predicates", "sbdt_gpu_microbench",
]


def lib_path() -> str:
    return os.path.join(_HERE, "libsbdt_gpu.so")


def lib():
    global _lib
    if _lib is None:
        path = lib_path()
        if not os.path.exists(path):
            raise SbdtGpuError(f"{path} missing: the CUDA extension is not built (run __graft_entry__.build())")
        L = C.CDLL(path)
        vp, u64, u32, u32p, u64p, dp, i8p, u8p = (C.c_void_p, C.c_uint64, C.c_uint32, C.POINTER(C.c_uint32),
                                                  C.POINTER(C.c_uint64), C.POINTER(C.c_double), C.POINTER(C.c_int8),
                                                  C.POINTER(C.c_uint8))
        L.sbdt_gpu_host_alloc.argtypes = [C.c_uint64, C.POINTER(vp)]
        L.sbdt_gpu_host_free.argtypes = [vp]
        L.sbdt_gpu_host_free.restype = None
        L.sbdt_gpu_create.argtypes = [C.c_int, C.POINTER(vp)]
        L.sbdt_gpu_destroy.argtypes = [vp]
        L.sbdt_gpu_destroy.restype = None
        L.sbdt_gpu_last_error.argtypes = [vp]
        L.sbdt_gpu_last_error.restype = C.c_char_p
        L.sbdt_gpu_set_stream.argtypes = [vp, vp]
        L.sbdt_gpu_synchronize.argtypes = [vp]
        L.sbdt_gpu_launch_count.argtypes = [vp]
        L.sbdt_gpu_launch_count.restype = C.c_ulonglong
        L.sbdt_gpu_check_status.argtypes = [vp]
        L.sbdt_gpu_assign_points.argtypes = [vp, C.c_int, dp, u64, u32p, u32p, u32, u32, u32p, u64p, u32p, dp]
        L.sbdt_gpu_assign_points_dev.argtypes = [vp, C.c_int, vp, u64, vp, vp, u32, u32, vp, vp, vp, vp]
        L.sbdt_gpu_find_border.argtypes = [vp, C.c_int, dp, u64, u32p, u32, u64p, u32p, u32p, i8p, C.c_int, C.c_double,
                                           u32, u8p, u8p, u32p, u64p, u32p, u64p, dp, dp, u64]
        L.sbdt_gpu_find_border_dev.argtypes = [vp, C.POINTER(BorderArgs)]
        L.sbdt_gpu_merge.argtypes = [vp, C.c_int, u32p, u64, u32, u64p, u32p, u32p, i8p, u8p, u32p, u32p, i8p, u64,
                                     u32, u64, u32p, u32p, i8p, u64p, u64p]
        L.sbdt_gpu_merge_dev.argtypes = [vp, C.POINTER(MergeArgs), u64, vp, vp, vp, vp, u64p]
        L.sbdt_gpu_set_timing.argtypes = [vp, C.c_int]
        L.sbdt_gpu_stage_times.argtypes = [vp, C.c_char_p, C.c_int, C.POINTER(C.c_float), C.c_int]
        L.sbdt_gpu_assign_table_stats.argtypes = [vp, C.POINTER(C.c_uint)]
        L.sbdt_gpu_border_stats.argtypes = [vp, C.POINTER(C.c_ulonglong), C.c_int]
        L.sbdt_gpu_predicates.argtypes = [vp, C.c_int, C.c_int, dp, u64, i8p, u64p]
        L.sbdt_gpu_microbench.argtypes = [vp, C.c_int, u64, dp]
        _lib = L
    return _lib


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


class Context:
    """One device context (stream + workspace) per host thread."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        rc = lib().sbdt_gpu_create(device, C.byref(self._h))
        if rc != SBDT_OK:
            raise SbdtGpuError(f"sbdt_gpu_create(device={device}) failed with status {rc} (no CUDA device?)")

    @property
    def handle(self):
        return self._h

    def check(self, rc: int, what: str):
        if rc == SBDT_OK:
            return
        msg = lib().sbdt_gpu_last_error(self._h).decode()
        if rc == SBDT_ERR_DEGENERATE:
            raise DegenerateSimplex(msg)
        if rc == SBDT_ERR_INVALID:
            raise ValueError(f"{what}: {msg}")
        if rc == SBDT_ERR_MERGE:
            raise InconsistentMerge(f"{what}: {msg}")
        raise SbdtGpuError(f"{what}: status {rc}: {msg}")

    def set_stream(self, stream_handle: int | None):
        self.check(lib().sbdt_gpu_set_stream(self._h, C.c_void_p(stream_handle or 0)), "set_stream")

    def synchronize(self):
        self.check(lib().sbdt_gpu_synchronize(self._h), "synchronize")

    @property
    def launches(self) -> int:
        return int(lib().sbdt_gpu_launch_count(self._h))

    def set_timing(self, enable: bool, census: bool = False):
        """Per-stage CUDA-event timing; census=True also fills the pipeline
        counters (table_stats / border_stats) at the cost of extra atomics."""
        self.check(lib().sbdt_gpu_set_timing(self._h, (1 if enable else 0) | (2 if census else 0)), "set_timing")

    def stage_times(self) -> list[tuple[str, float]]:
        """(stage, ms) pairs recorded since the last call (CUDA events on the context stream)."""
        names = C.create_string_buffer(1 << 16)
        ms = (C.c_float * 4096)()
        cnt = lib().sbdt_gpu_stage_times(self._h, names, 1 << 16, ms, 4096)
        if cnt < 0:
            self.check(-cnt, "stage_times")
        labels = names.value.decode().split("\n")[:cnt]
        return [(labels[i], float(ms[i])) for i in range(cnt)]

    def table_stats(self) -> dict:
        out = (C.c_uint * 6)()
        if lib().sbdt_gpu_assign_table_stats(self._h, out) != SBDT_OK:
            return {}
        return {"uniform": int(out[0]), "list": int(out[1]), "ring_search": int(out[2]), "long_list": int(out[3]),
                "queued_points": int(out[4]), "dense_cells": int(out[5])}

    def border_stats(self) -> dict:
        out = (C.c_ulonglong * 20)()
        if lib().sbdt_gpu_border_stats(self._h, out, 20) != SBDT_OK:
            return {}
        keys = {0: "rows", 1: "exact_stage_rows", 2: "exact_flat_scan", 3: "wide_from_exact", 4: "wide_rows",
                5: "row_pairs", 6: "wide_expansions", 7: "exact_flat_positive", 8: "prefilter_positive",
                9: "wide_positive", 10: "mask_positive", 12: "orient_check_rows", 13: "orient_escalations",
                14: "in_sphere_escalations", 15: "mask_negative", 16: "scan32_rows", 17: "scan32_positive",
                18: "scan32_open"}
        return {kk: int(out[i]) for i, kk in keys.items()}

    # ---- diagnostics (tests / bench): device predicates, binding ceilings
    def predicates(self, op: str, pts: np.ndarray):
        """Device orient / in_sphere (filter + expansion arithmetic) on host
        cases: pts (count, dim+1, dim) for "orient", (count, dim+2, dim) for
        "in_sphere" (simplex then q). Returns (signs int8, n_escalated)."""
        pts = np.ascontiguousarray(pts, np.float64)
        count, npts, dim = pts.shape
        opc = {"orient": 0, "in_sphere": 1}[op]
        if npts != dim + 1 + opc:
            raise ValueError("predicates: wrong point count per case")
        out = np.empty(count, np.int8)
        ne = C.c_uint64(0)
        self.check(lib().sbdt_gpu_predicates(self._h, opc, dim, _p(pts, C.c_double), count, _p(out, C.c_int8),
                                             C.byref(ne)), "predicates")
        return out, int(ne.value)

    def microbench(self, kind: str, nbytes: int = 0) -> float:
        """"dfma" -> FLOP/s; "gather" -> random 8-byte gathers/s from an nbytes table."""
        r = C.c_double(0)
        self.check(lib().sbdt_gpu_microbench(self._h, {"dfma": 0, "gather": 1}[kind], nbytes, C.byref(r)),
                   "microbench")
        return float(r.value)

    # ---- device-pointer entry points (inputs resident in HBM; async on the stream)
    def assign_points_dev(self, dim, d_xyz, n, d_sample_ids, d_sample_labels, m, k, d_labels, d_part_offsets=None,
                          d_part_ids=None, d_bbox=None):
        rc = lib().sbdt_gpu_assign_points_dev(self._h, dim, d_xyz, n, d_sample_ids, d_sample_labels, m, k, d_labels,
                                              d_part_offsets, d_part_ids, d_bbox)
        self.check(rc, "assign_points_dev")

    def find_border_dev(self, args: "BorderArgs"):
        self.check(lib().sbdt_gpu_find_border_dev(self._h, C.byref(args)), "find_border_dev")

    def merge_dev(self, args: "MergeArgs", capacity: int, d_out_verts, d_out_nbrs, d_out_parity, d_out_offsets) -> int:
        """Device-pointer merge (outputs with row stride `capacity`); returns the row count."""
        rows = C.c_uint64(0)
        self.check(lib().sbdt_gpu_merge_dev(self._h, C.byref(args), capacity, d_out_verts, d_out_nbrs, d_out_parity,
                                            d_out_offsets, C.byref(rows)), "merge_dev")
        return int(rows.value)

    def close(self):
        if self._h:
            lib().sbdt_gpu_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Context | None = None


class _PinnedBlock:
    """Owner of one sbdt_gpu_host_alloc block (freed with the last view)."""

    def __init__(self, nbytes: int):
        self.ptr = C.c_void_p()
        rc = lib().sbdt_gpu_host_alloc(max(int(nbytes), 1), C.byref(self.ptr))
        if rc != SBDT_OK:
            raise MemoryError(f"sbdt_gpu_host_alloc({nbytes}) failed with status {rc}")

    def __del__(self):
        if getattr(self, "ptr", None) and self.ptr.value:
            lib().sbdt_gpu_host_free(self.ptr)
            self.ptr = C.c_void_p()


def pinned_empty(shape, dtype) -> np.ndarray:
    """Page-locked numpy array for the host-buffer entry points' inputs and
    outputs (pageable buffers are staged by the driver and fault in fresh pages)."""
    dtype = np.dtype(dtype)
    shape = (shape,) if np.isscalar(shape) else tuple(shape)
    nbytes = int(np.prod(shape, dtype=np.int64)) * dtype.itemsize
    blk = _PinnedBlock(nbytes)
    buf = (C.c_char * max(nbytes, 1)).from_address(blk.ptr.value)
    buf._owner = blk  # keep the block alive as long as any view
    return np.frombuffer(buf, dtype=dtype, count=nbytes // dtype.itemsize).reshape(shape)


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


@dataclass
class Partitioning:
    """labels, parts (CSR: parts_offsets, parts_ids), sample ids/labels."""
    labels: np.ndarray
    parts_offsets: np.ndarray
    parts_ids: np.ndarray
    sample_point_ids: np.ndarray
    sample_labels: np.ndarray
    bbox: np.ndarray

    def part(self, i: int) -> np.ndarray:
        return self.parts_ids[self.parts_offsets[i]:self.parts_offsets[i + 1]]


def _out(buf, shape, dtype):
    if buf is None:
        return np.empty(shape, dtype)
    if buf.dtype != np.dtype(dtype) or buf.shape != ((shape,) if np.isscalar(shape) else tuple(shape)) \
            or not buf.flags.c_contiguous:
        raise ValueError(f"output buffer must be a contiguous {np.dtype(dtype)} array of shape {shape}")
    return buf


def assign_points(points: np.ndarray, sample_ids: np.ndarray, sample_labels: np.ndarray, k: int,
                  ctx: Context | None = None, out: Partitioning | None = None) -> Partitioning:
    """assign_points through the host-buffer C ABI entry point.
    `out` (optional): a Partitioning whose labels / parts_offsets / parts_ids /
    bbox arrays are reused as output buffers (e.g. pinned_empty arrays)."""
    ctx = ctx or default_context()
    pts = np.ascontiguousarray(points, np.float64)
    n, dim = pts.shape
    sid = np.ascontiguousarray(sample_ids, np.uint32)
    slab = np.ascontiguousarray(sample_labels, np.uint32)
    labels = _out(out.labels if out else None, n, np.uint32)
    poff = _out(out.parts_offsets if out else None, k + 1, np.uint64)
    pids = _out(out.parts_ids if out else None, n, np.uint32)
    bbox = _out(out.bbox if out else None, 2 * dim, np.float64)
    rc = lib().sbdt_gpu_assign_points(ctx.handle, dim, _p(pts, C.c_double), n, _p(sid, C.c_uint32),
                                      _p(slab, C.c_uint32), len(sid), k, _p(labels, C.c_uint32),
                                      _p(poff, C.c_uint64), _p(pids, C.c_uint32), _p(bbox, C.c_double))
    ctx.check(rc, "assign_points")
    return Partitioning(labels, poff, pids, sid, slab, bbox)


@dataclass
class IntersectionPolicy:
    """kind in {bbox, grid, exact}, c_G > 0."""
    kind: str = "grid"
    c_G: float = 1.0


@dataclass
class BorderSet:
    """SPEC.md:472-476 plus the north_star full-scan flags."""
    positive: np.ndarray              # per simplex row: full-scan positive flag
    border: np.ndarray | None         # per simplex row: SPEC BFS border flag
    border_vertex_ids: np.ndarray     # vertices(border) (SPEC BorderSet), sorted
    positive_vertex_ids: np.ndarray   # vertices(positive) (north_star), sorted
    spheres: np.ndarray | None = None

    def simplex_ids(self, partials, part: int, which: str = "border") -> np.ndarray:
        flags = self.border if which == "border" else self.positive
        lo, hi = int(partials.offsets[part]), int(partials.offsets[part + 1])
        return np.nonzero(flags[lo:hi])[0].astype(np.uint32)


def find_border(points: np.ndarray, labels: np.ndarray, partials, policy: IntersectionPolicy | None = None,
                hull_bfs: bool = True, spheres: bool = False, ctx: Context | None = None,
                out: BorderSet | None = None, resident: bool = False, grid_bbox=None,
                grid_n_total: int = 0) -> BorderSet:
    """find_border through the host-buffer C ABI entry point.
    `out` (optional): a BorderSet whose positive / border arrays (length S) and
    border_vertex_ids / positive_vertex_ids arrays (length n) are reused as
    output buffers; the result then holds views into them. resident=True:
    `points` and `labels` are the arrays of the last assign_points call on
    `ctx` (labels = its Partitioning.labels), unchanged: their device copies
    are reused instead of uploaded (SBDT_BORDER_RESIDENT_POINTS).
    Recursion levels: grid_bbox (lo, hi) and grid_n_total
    give the top level's grid (GridIndex global bbox / n_total); points
    outside the level carry the label UNINDEXED."""
    ctx = ctx or default_context()
    policy = policy or IntersectionPolicy()
    pts = np.ascontiguousarray(points, np.float64)
    n, dim = pts.shape
    lab = np.ascontiguousarray(labels, np.uint32)
    S, k = partials.S, partials.k
    pos = _out(out.positive if out else None, S, np.uint8)
    bor = _out(out.border if out else None, S, np.uint8) if hull_bfs else None
    vids = _out(out.positive_vertex_ids if out else None, n, np.uint32)
    bvids = _out(out.border_vertex_ids if out else None, n, np.uint32) if hull_bfs else None
    nv, nb = C.c_uint64(0), C.c_uint64(0)
    sph = np.empty((S, dim + 1), np.float64) if spheres else None
    gbb = None if grid_bbox is None else np.ascontiguousarray(np.concatenate([np.asarray(grid_bbox[0], np.float64),
                                                                              np.asarray(grid_bbox[1], np.float64)]))
    rc = lib().sbdt_gpu_find_border(
        ctx.handle, dim, _p(pts, C.c_double), n, _p(lab, C.c_uint32), k, _p(partials.offsets, C.c_uint64),
        _p(partials.verts, C.c_uint32), _p(partials.nbrs, C.c_uint32), _p(partials.parity, C.c_int8),
        POLICY[policy.kind], policy.c_G, (HULL_BFS if hull_bfs else 0) | (RESIDENT_POINTS if resident else 0),
        _p(pos, C.c_uint8),
        _p(bor, C.c_uint8) if hull_bfs else None, _p(vids, C.c_uint32), C.byref(nv),
        _p(bvids, C.c_uint32) if hull_bfs else None, C.byref(nb) if hull_bfs else None,
        _p(sph, C.c_double) if spheres else None,
        _p(gbb, C.c_double) if gbb is not None else None, int(grid_n_total))
    ctx.check(rc, "find_border")
    if out is not None:  # views into the caller's buffers
        return BorderSet(pos, bor, bvids[:nb.value] if hull_bfs else vids[:nv.value], vids[:nv.value], sph)
    return BorderSet(pos, bor, bvids[:nb.value].copy() if hull_bfs else vids[:nv.value].copy(),
                     vids[:nv.value].copy(), sph)


@dataclass
class Merged:
    """The merged triangulation, vertex-major SoA like host.Tri.
    offsets (k+3): rows of part p are [offsets[p], offsets[p+1]); the inserted
    T_B rows [offsets[k], offsets[k+1]); the hull rows [offsets[k+1], offsets[k+2])."""
    verts: np.ndarray   # (D+1, R) uint32
    nbrs: np.ndarray    # (D+1, R) uint32
    parity: np.ndarray  # (R,) int8
    offsets: np.ndarray  # (k+3,) uint64


def merge(partials, border: np.ndarray, tb, labels: np.ndarray, hull: bool = True,
          ctx: Context | None = None) -> Merged:
    """merge + update_neighbors through the host-buffer C ABI.
    `border`: per partial row, nonzero = border simplex (BorderSet.border or
    .positive); `tb`: the triangulation of the border vertices (host.Tri:
    verts / nbrs (D+1, S_B), parity); `labels`: the partition of every point.
    hull=True appends the re-derived infinite simplices (reference layout);
    False leaves kNone links on the hull facets."""
    ctx = ctx or default_context()
    dim = partials.verts.shape[0] - 1
    k, S = partials.k, partials.S
    bor = np.ascontiguousarray(border, np.uint8)
    if bor.shape != (S,):
        raise ValueError("merge: border must hold one flag per partial row")
    lab = np.ascontiguousarray(labels, np.uint32)
    tv = np.ascontiguousarray(tb.verts, np.uint32)
    tn = np.ascontiguousarray(tb.nbrs, np.uint32)
    tp = np.ascontiguousarray(tb.parity, np.int8)
    SB = tv.shape[1]
    cap = S + SB + 64
    for _ in range(3):
        ov = np.empty((dim + 1) * cap, np.uint32)
        on = np.empty((dim + 1) * cap, np.uint32)
        op = np.empty(cap, np.int8)
        oo = np.empty(k + 3, np.uint64)
        rows = C.c_uint64(0)
        rc = lib().sbdt_gpu_merge(ctx.handle, dim, _p(lab, C.c_uint32), len(lab), k, _p(partials.offsets, C.c_uint64),
                                  _p(partials.verts, C.c_uint32), _p(partials.nbrs, C.c_uint32),
                                  _p(partials.parity, C.c_int8), _p(bor, C.c_uint8), _p(tv, C.c_uint32),
                                  _p(tn, C.c_uint32), _p(tp, C.c_int8), SB, MERGE_HULL if hull else 0, cap,
                                  _p(ov, C.c_uint32), _p(on, C.c_uint32), _p(op, C.c_int8), _p(oo, C.c_uint64),
                                  C.byref(rows))
        if rc == SBDT_ERR_RANGE and rows.value > cap:
            cap = int(rows.value) * 2 + 64
            continue
        ctx.check(rc, "merge")
        R = int(rows.value)
        return Merged(ov[:(dim + 1) * R].reshape(dim + 1, R), on[:(dim + 1) * R].reshape(dim + 1, R), op[:R], oo)
    raise SbdtGpuError("merge: output capacity retry failed")
