"""TEST INFRASTRUCTURE — full-size parity of one GPU run against the CPU
oracle (used by tests/test_gpu_fullsize.py and bench.py's parity leg).

Ground truth, per SPEC.md:
  labels      assign_points = nearest sample by squared_distance, ties to the
              lowest sample PointId (the kd-tree oracle equals
              brute force, pinned in tests/test_oracle.py)
  parts       Partitioning.parts = the point ids of each part, ascending
              (SPEC.md:307-312, :382): a stable counting sort of the labels
  positive    north_star full scan: some occupied cell of another part
              overlaps the inflated circumsphere / outer halfspace
              
  border      SPEC find_border BFS from hull_simplices
  vertex sets sorted unique finite vertices of positive / border rows
"""
from __future__ import annotations

import time

import numpy as np

from . import assign_kdtree, find_border


def oracle_parts(labels: np.ndarray, k: int):
    lab = np.asarray(labels)
    counts = np.bincount(lab, minlength=k).astype(np.uint64)
    offsets = np.zeros(k + 1, np.uint64)
    np.cumsum(counts, out=offsets[1:])
    ids = np.argsort(lab, kind="stable").astype(np.uint32)
    return offsets, ids


def _first_diff(a, b):
    if a.shape != b.shape:
        return f"shape {a.shape} vs {b.shape}"
    idx = np.flatnonzero(a != b)
    return f"{len(idx)} differ, first at {int(idx[0])}: {a[idx[0]]} vs {b[idx[0]]}" if len(idx) else None


def check_labels(points, sample_ids, sample_labels, k, labels, parts_offsets=None, parts_ids=None, threads=8):
    """Oracle labels (kd-tree, all `threads`) vs the GPU's; returns (result dict, oracle labels)."""
    t0 = time.perf_counter()
    ref = assign_kdtree(points, sample_ids, sample_labels, threads)
    t_assign = time.perf_counter() - t0
    res = {"labels": _first_diff(np.asarray(labels), ref) is None, "assign_s": round(t_assign, 3)}
    if res["labels"] is False:
        res["labels_diff"] = _first_diff(np.asarray(labels), ref)
    if parts_offsets is not None:
        off, ids = oracle_parts(ref, k)
        res["parts"] = bool(np.array_equal(np.asarray(parts_offsets, np.uint64), off)
                            and np.array_equal(np.asarray(parts_ids, np.uint32), ids))
    return res, ref


def check_border(points, labels, partials, positive, border, positive_vertex_ids, border_vertex_ids,
                 policy="grid", threads=8):
    """Oracle find_border (full scan + BFS, all `threads`) vs the GPU's outputs.
    `border` / `border_vertex_ids` may be None (no-BFS run)."""
    o = find_border(points, labels, partials, policy, threads=threads)
    res = {"positive": bool(np.array_equal(np.asarray(positive), o["positive"])),
           "positive_vertices": bool(np.array_equal(np.asarray(positive_vertex_ids), o["vertices_positive"])),
           "index_build_s": round(o["times"][0], 3), "border_s": round(o["times"][1], 3),
           "n_positive": int(o["positive"].sum()), "n_border": int(o["border"].sum()),
           "n_positive_vertices": len(o["vertices_positive"]), "n_border_vertices": len(o["vertices_border"])}
    if not res["positive"]:
        res["positive_diff"] = _first_diff(np.asarray(positive), o["positive"])
    if border is not None:
        res["border"] = bool(np.array_equal(np.asarray(border), o["border"]))
        res["border_vertices"] = bool(np.array_equal(np.asarray(border_vertex_ids), o["vertices_border"]))
    return res


def all_equal(res: dict) -> bool:
    keys = ("labels", "parts", "positive", "positive_vertices", "border", "border_vertices")
    return all(res[k] for k in keys if k in res)
