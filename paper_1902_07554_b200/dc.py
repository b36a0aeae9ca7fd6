"""One level of Alg. 1 (dc-engine `delaunay_dc`) with the
k-way strategy, composed from the GPU path and the host setup:

  draw_sample + partition (host)  ->  assign_points (GPU)  ->  k partial DTs
  (host)  ->  find_border (GPU)  ->  T_B = DT of the border vertices (host)
  ->  merge + update_neighbors (GPU)

The partial and border triangulations are host setup (the sequential DT
builder, not on the data-parallel path); the recursion of SPEC.md's
delaunay_dc is not built. For general-position inputs the result equals the
sequential DT of the whole point set (the master property).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import gpu, host


@dataclass
class DcResult:
    merged: gpu.Merged
    labels: np.ndarray
    partials: host.Partials
    border: gpu.BorderSet
    tb: host.Tri


def delaunay_dc_once(points: np.ndarray, k: int, seed: int = 1, frac: float = 0.01,
                     policy: gpu.IntersectionPolicy | None = None, border: str = "bfs", hull: bool = True,
                     ctx: gpu.Context | None = None) -> DcResult:
    """border: "bfs" (SPEC find_border, hull-reachable) or "positive" (every
    positive simplex, the north_star's full scan)."""
    ctx = ctx or gpu.default_context()
    pts = np.ascontiguousarray(points, np.float64)
    n = len(pts)
    m = max(pts.shape[1] + 2, int(round(frac * n)))
    sid = host.draw_sample(n, m, seed)
    slab, _ = host.partition_sample(pts, sid, k, seed)
    part = gpu.assign_points(pts, sid, slab, k, ctx=ctx)
    partials = host.build_partials(pts, part.labels, k, seed)
    bs = gpu.find_border(pts, part.labels, partials, policy, hull_bfs=True, ctx=ctx)
    flags, vids = (bs.border, bs.border_vertex_ids) if border == "bfs" else (bs.positive, bs.positive_vertex_ids)
    if len(vids) >= pts.shape[1] + 1:
        tb = host.triangulate(pts, vids, seed)
    else:
        tb = host.Tri(np.zeros((pts.shape[1] + 1, 0), np.uint32), np.zeros((pts.shape[1] + 1, 0), np.uint32),
                      np.zeros(0, np.int8))
    merged = gpu.merge(partials, flags, tb, part.labels, hull=hull, ctx=ctx)
    return DcResult(merged, part.labels, partials, bs, tb)
