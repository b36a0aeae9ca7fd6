"""Host setup pipeline (ctypes over libsbdt_host.so).

Produces the hot path's inputs — seeded point sets, the sample, the sample's
k-way labels and the k partial Delaunay triangulations — exactly as SPEC.md's
partition_points / delaunay_dc would before calling assign_points and
find_border. Nothing here is on the measured GPU
path; it runs once per instance on the host.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None

DIST = {"uniform": 0, "normal": 1, "bubbles": 2, "lines": 3}
WEIGHTS = {"constant": 0, "inverse": 1, "log": 2, "linear": 3}


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "libsbdt_host.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build())")
        L = C.CDLL(path)
        u64, u32p, dp, i8p = C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_double), C.POINTER(C.c_int8)
        L.sbdt_host_generate.restype = u64
        L.sbdt_host_generate.argtypes = [C.c_int, C.c_int, u64, u64, dp, C.c_int, dp]
        L.sbdt_host_deduplicate.restype = u64
        L.sbdt_host_deduplicate.argtypes = [C.c_int, dp, u64, u32p]
        L.sbdt_host_draw_sample.argtypes = [u64, u64, u64, u32p]
        L.sbdt_host_triangulate.restype = C.c_void_p
        L.sbdt_host_triangulate.argtypes = [C.c_int, dp, u32p, u64, u64, C.c_char_p, C.c_int]
        L.sbdt_host_tri_count.restype = u64
        L.sbdt_host_tri_count.argtypes = [C.c_void_p]
        L.sbdt_host_tri_export.argtypes = [C.c_void_p, u32p, u32p, i8p]
        L.sbdt_host_tri_free.argtypes = [C.c_void_p]
        L.sbdt_host_partition_sample.argtypes = [C.c_int, dp, u32p, u64, C.c_uint32, C.c_double, C.c_int, u64,
                                                 u32p, C.POINTER(C.c_uint64), C.c_char_p, C.c_int]
        L.sbdt_host_partition_csr.argtypes = [u64, u32p, u32p, C.POINTER(C.c_int32), C.c_uint32, C.c_double, u64,
                                              u32p, C.POINTER(C.c_uint64), C.c_char_p, C.c_int]
        L.sbdt_host_build_partials.restype = C.c_void_p
        L.sbdt_host_build_partials.argtypes = [C.c_int, dp, u64, u32p, C.c_uint32, u64, C.c_int, C.c_char_p, C.c_int]
        L.sbdt_host_partials_total.restype = u64
        L.sbdt_host_partials_total.argtypes = [C.c_void_p]
        L.sbdt_host_partials_export.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), u32p, u32p, i8p]
        L.sbdt_host_partials_free.argtypes = [C.c_void_p]
        L.sbdt_host_predicates.argtypes = [C.c_int, C.c_int, dp, u64, C.POINTER(C.c_int8)]
        _lib = L
    return _lib


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def generate(dist: str, dim: int, n: int, seed: int, params=()) -> np.ndarray:
    out = np.empty(n * dim, dtype=np.float64)
    p = np.asarray(params, dtype=np.float64)
    got = lib().sbdt_host_generate(DIST[dist], dim, n, seed, ptr(p, C.c_double) if len(p) else None, len(p),
                                   ptr(out, C.c_double))
    if got != n:
        raise ValueError(f"generate({dist}, dim={dim}) failed")
    return out.reshape(n, dim)


def predicates(op: str, pts: np.ndarray) -> np.ndarray:
    """The shared predicates (predicates.hpp) on the host, same layout as
    gpu.Context.predicates: (count, dim+1, dim) orient / (count, dim+2, dim)
    in_sphere cases -> signs."""
    pts = np.ascontiguousarray(pts, np.float64)
    count, _, dim = pts.shape
    out = np.empty(count, np.int8)
    if lib().sbdt_host_predicates({"orient": 0, "in_sphere": 1}[op], dim, ptr(pts, C.c_double), count,
                                  ptr(out, C.c_int8)) != 0:
        raise ValueError("predicates: bad op / dim")
    return out


def deduplicate(points: np.ndarray) -> np.ndarray:
    pts = np.ascontiguousarray(points, dtype=np.float64).copy()
    n, dim = pts.shape
    m = lib().sbdt_host_deduplicate(dim, ptr(pts, C.c_double), n, None)
    return pts[:m].copy() if m != n else pts


def draw_sample(n: int, m: int, seed: int) -> np.ndarray:
    out = np.empty(m, dtype=np.uint32)
    if lib().sbdt_host_draw_sample(n, m, seed, ptr(out, C.c_uint32)) != 0:
        raise ValueError("draw_sample failed")
    return out


@dataclass
class Tri:
    """Compacted triangulation, vertex-major SoA (row j = vertices[j] of every simplex)."""
    verts: np.ndarray   # (D+1, S) uint32
    nbrs: np.ndarray    # (D+1, S) uint32
    parity: np.ndarray  # (S,) int8


def triangulate(points: np.ndarray, ids: np.ndarray, seed: int) -> Tri:
    pts = np.ascontiguousarray(points, dtype=np.float64)
    dim = pts.shape[1]
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    err = C.create_string_buffer(256)
    h = lib().sbdt_host_triangulate(dim, ptr(pts, C.c_double), ptr(ids, C.c_uint32), len(ids), seed, err, 256)
    if not h:
        raise ValueError("triangulate: " + err.value.decode())
    try:
        S = lib().sbdt_host_tri_count(h)
        v = np.empty((dim + 1, S), np.uint32)
        nb = np.empty((dim + 1, S), np.uint32)
        par = np.empty(S, np.int8)
        lib().sbdt_host_tri_export(h, ptr(v, C.c_uint32), ptr(nb, C.c_uint32), ptr(par, C.c_int8))
    finally:
        lib().sbdt_host_tri_free(h)
    return Tri(v, nb, par)


def partition_sample(points: np.ndarray, sample_ids: np.ndarray, k: int, seed: int, eps: float = 0.05,
                     weights: str = "log"):
    pts = np.ascontiguousarray(points, dtype=np.float64)
    sid = np.ascontiguousarray(sample_ids, dtype=np.uint32)
    labels = np.empty(len(sid), np.uint32)
    cut = C.c_uint64(0)
    err = C.create_string_buffer(256)
    rc = lib().sbdt_host_partition_sample(pts.shape[1], ptr(pts, C.c_double), ptr(sid, C.c_uint32), len(sid), k, eps,
                                          WEIGHTS[weights], seed, ptr(labels, C.c_uint32), C.byref(cut), err, 256)
    if rc != 0:
        raise ValueError("partition_sample: " + err.value.decode())
    return labels, int(cut.value)


def partition_csr(xadj, adj, w, k: int, eps: float = 0.05, seed: int = 1):
    xadj = np.ascontiguousarray(xadj, np.uint32)
    adj = np.ascontiguousarray(adj, np.uint32)
    w = np.ascontiguousarray(w, np.int32)
    n = len(xadj) - 1
    labels = np.empty(n, np.uint32)
    cut = C.c_uint64(0)
    err = C.create_string_buffer(256)
    rc = lib().sbdt_host_partition_csr(n, ptr(xadj, C.c_uint32), ptr(adj, C.c_uint32), ptr(w, C.c_int32), k, eps,
                                       seed, ptr(labels, C.c_uint32), C.byref(cut), err, 256)
    if rc != 0:
        raise ValueError(err.value.decode())
    return labels, int(cut.value)


@dataclass
class Partials:
    """k partial DTs concatenated: part p owns simplex rows [offsets[p], offsets[p+1])."""
    offsets: np.ndarray  # (k+1,) uint64
    verts: np.ndarray    # (D+1, S) uint32, global point ids
    nbrs: np.ndarray     # (D+1, S) uint32, part-local simplex ids
    parity: np.ndarray   # (S,) int8

    @property
    def k(self) -> int:
        return len(self.offsets) - 1

    @property
    def S(self) -> int:
        return int(self.offsets[-1])


def build_partials(points: np.ndarray, labels: np.ndarray, k: int, seed: int, threads: int = 0) -> Partials:
    pts = np.ascontiguousarray(points, dtype=np.float64)
    lab = np.ascontiguousarray(labels, dtype=np.uint32)
    dim = pts.shape[1]
    err = C.create_string_buffer(256)
    h = lib().sbdt_host_build_partials(dim, ptr(pts, C.c_double), len(pts), ptr(lab, C.c_uint32), k, seed, threads,
                                       err, 256)
    if not h:
        raise ValueError("build_partials: " + err.value.decode())
    try:
        S = lib().sbdt_host_partials_total(h)
        off = np.empty(k + 1, np.uint64)
        v = np.empty((dim + 1, S), np.uint32)
        nb = np.empty((dim + 1, S), np.uint32)
        par = np.empty(S, np.int8)
        lib().sbdt_host_partials_export(h, ptr(off, C.c_uint64), ptr(v, C.c_uint32), ptr(nb, C.c_uint32),
                                        ptr(par, C.c_int8))
    finally:
        lib().sbdt_host_partials_free(h)
    return Partials(off, v, nb, par)


# ---------------------------------------------------------------------------
# BASELINE.json configs. n is overridable for test-scale runs.
# ---------------------------------------------------------------------------
CONFIGS = {
    1: dict(name="cfg1-2d-uniform-1M", dist="uniform", dim=2, n=1_000_000, seed=1, frac=0.01, k=16),
    2: dict(name="cfg2-3d-uniform-10M", dist="uniform", dim=3, n=10_000_000, seed=2, frac=0.01, k=64),
    3: dict(name="cfg3-3d-normal-10M", dist="normal", dim=3, n=10_000_000, seed=3, frac=0.01, k=64),
    4: dict(name="cfg4-3d-bubbles-20M", dist="bubbles", dim=3, n=20_000_000, seed=4, frac=0.005, k=128),
    5: dict(name="cfg5-2d-lines-50M", dist="lines", dim=2, n=50_000_000, seed=5, frac=0.002, k=256),
}


@dataclass
class Instance:
    config: dict
    points: np.ndarray
    sample_ids: np.ndarray
    sample_labels: np.ndarray
    cut: int = 0
    labels: np.ndarray | None = None
    partials: Partials | None = None
    timings: dict = field(default_factory=dict)

    @property
    def dim(self):
        return self.points.shape[1]

    @property
    def n(self):
        return self.points.shape[0]


def make_instance(cfg: int | dict, n: int | None = None, k: int | None = None, seed: int | None = None,
                  frac: float | None = None) -> Instance:
    """Generate points, deduplicate, draw the sample and partition the sample DT."""
    import time
    c = dict(CONFIGS[cfg]) if isinstance(cfg, int) else dict(cfg)
    if n is not None:
        c["n"] = n
    if k is not None:
        c["k"] = k
    if seed is not None:
        c["seed"] = seed
    if frac is not None:
        c["frac"] = frac
    t0 = time.time()
    pts = generate(c["dist"], c["dim"], c["n"], c["seed"])
    pts = deduplicate(pts)
    t1 = time.time()
    m = max(c["dim"] + 2, int(round(c["frac"] * len(pts))))
    sid = draw_sample(len(pts), m, c["seed"])
    slab, cut = partition_sample(pts, sid, c["k"], c["seed"])
    t2 = time.time()
    inst = Instance(c, pts, sid, slab, cut)
    inst.timings.update(generate_s=t1 - t0, sample_partition_s=t2 - t1)
    return inst


def attach_partials(inst: Instance, labels: np.ndarray, threads: int = 0) -> Partials:
    import time
    t0 = time.time()
    inst.labels = labels
    inst.partials = build_partials(inst.points, labels, inst.config["k"], inst.config["seed"], threads)
    inst.timings["partials_s"] = time.time() - t0
    return inst.partials
