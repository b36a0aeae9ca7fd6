#!/usr/bin/env python3
"""Benchmark of the merge + update_neighbors step (SURVEY.md
§8f row 4) on one B200 — the step after the border triangulation.

Setup (untimed): the BASELINE config's points, sample partition, labels
(GPU assign_points), the k partial DTs and the border flags (GPU find_border),
and T_B = the DT of the border vertices (host builder). One step = one merge
of the k partials with T_B (keep / include bitmaps, scan, emission with the
facet-hash join, hull re-derivation), inputs resident in HBM; e2e = the same
through the host-buffer C ABI (sbdt_gpu_merge) from page-locked buffers.

  python tools/bench_merge.py [--config 2] [--steps 5] [--warmup 3] [--border bfs|positive]

Prints one JSON line; metric = simplex rows merged per second, rows = the
partial rows plus the T_B rows the step consumes.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--border", default="bfs", choices=["bfs", "positive"])
    ap.add_argument("--cpu-n", type=int, default=400_000, help="points of the oracle's bounded sample instance")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    import torch
    import bench
    from paper_1902_07554_b200 import gpu, host

    dev = torch.device("cuda", 0)
    t0 = time.time()
    inst = host.make_instance(args.config, n=args.n, k=args.k)
    dim, n, k = inst.dim, inst.n, inst.config["k"]
    ctx = gpu.Context(0)
    part = gpu.assign_points(inst.points, inst.sample_ids, inst.sample_labels, k, ctx=ctx)
    P = host.attach_partials(inst, part.labels)
    bs = gpu.find_border(inst.points, part.labels, P, hull_bfs=True, ctx=ctx)
    flags, vids = (bs.border, bs.border_vertex_ids) if args.border == "bfs" else (bs.positive, bs.positive_vertex_ids)
    t1 = time.time()
    tb = host.triangulate(inst.points, vids, 1)
    t_tb = time.time() - t1
    setup_s = time.time() - t0
    S, SB = P.S, tb.verts.shape[1]

    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    d_lab = T(part.labels.view(np.int32))
    d_off = T(P.offsets.view(np.int64))
    d_v, d_n, d_p, d_b = T(P.verts.view(np.int32)), T(P.nbrs.view(np.int32)), T(P.parity), T(flags.astype(np.uint8))
    d_tv, d_tn, d_tp = T(tb.verts.view(np.int32)), T(tb.nbrs.view(np.int32)), T(tb.parity)
    cap = S + SB + 64
    d_ov = torch.empty((dim + 1) * cap, dtype=torch.int32, device=dev)
    d_on = torch.empty((dim + 1) * cap, dtype=torch.int32, device=dev)
    d_op = torch.empty(cap, dtype=torch.int8, device=dev)
    d_oo = torch.empty(k + 3, dtype=torch.int64, device=dev)
    a = gpu.MergeArgs()
    a.dim, a.k, a.d_labels, a.n, a.d_offsets = dim, k, d_lab.data_ptr(), n, d_off.data_ptr()
    a.d_verts, a.d_nbrs, a.d_parity, a.S, a.d_border = d_v.data_ptr(), d_n.data_ptr(), d_p.data_ptr(), S, d_b.data_ptr()
    a.d_tb_verts, a.d_tb_nbrs, a.d_tb_parity, a.S_B = d_tv.data_ptr(), d_tn.data_ptr(), d_tp.data_ptr(), SB
    a.flags = gpu.MERGE_HULL

    def step():
        return ctx.merge_dev(a, cap, d_ov.data_ptr(), d_on.data_ptr(), d_op.data_ptr(), d_oo.data_ptr())

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        rows = step()
    torch.cuda.synchronize()
    ctx.set_timing(True)
    ms, stages = [], {}
    l0 = ctx.launches
    with bench.ClockSampler(0) as clk:
        for _ in range(args.steps):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            rows = step()
            e.record(stream)
            e.synchronize()
            ms.append(s.elapsed_time(e))
            for name, t in ctx.stage_times():
                stages.setdefault(name, []).append(t)
    ctx.set_timing(False)
    launches = (ctx.launches - l0) // max(1, args.steps)
    step_ms = sum(ms) / len(ms)
    off = d_oo.cpu().numpy()
    M, H = int(off[k + 1]), int(off[k + 2] - off[k + 1])

    # e2e: host-buffer C ABI from page-locked buffers (H2D + merge + D2H)
    pin = lambda x: _pinned_copy(gpu, x)  # noqa: E731
    Pp = host.Partials(pin(P.offsets), pin(P.verts), pin(P.nbrs), pin(P.parity))
    tbp = host.Tri(pin(tb.verts), pin(tb.nbrs), pin(tb.parity))
    fl, lb = pin(flags.astype(np.uint8)), pin(part.labels)
    gpu.merge(Pp, fl, tbp, lb, ctx=ctx)
    e2e = []
    for _ in range(max(2, args.steps // 2)):
        t = time.perf_counter()
        gpu.merge(Pp, fl, tbp, lb, ctx=ctx)
        e2e.append(time.perf_counter() - t)
    e2e_s = min(e2e)
    D1 = dim + 1
    h2d = 8 * (k + 1) + S * (8 * D1 + 2) + SB * (8 * D1 + 1) + 4 * n
    d2h = rows * (8 * D1 + 1) + 8 * (k + 3)

    # algorithmic HBM bytes of one step: partial rows (verts, nbrs, parity,
    # border) and T_B rows read once, output rows written once, the T_B label
    # gathers (4 B per vertex) and the bitmaps
    alg = S * (8 * D1 + 2) + SB * (8 * D1 + 1 + 4 * D1) + rows * (8 * D1 + 1)
    peak, peak_kind = bench.peaks()
    ach = alg / (step_ms * 1e-3) / 1e9
    in_rows = S + SB
    line = {
        "metric": "simplex rows merged/s (partial + border-triangulation rows, merge + update_neighbors) on 1 B200",
        "value": in_rows / (step_ms * 1e-3), "unit": "rows/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded, BASELINE.json config)",
        "config": {"workload": inst.config["name"] + "-merge", "n": n, "k": k, "S": S, "S_B": SB,
                   "border": args.border, "rows_out": rows, "finite_out": M, "hull_rows": H,
                   "l2": "flushed (256 MB write) before every step", "setup_s": round(setup_s, 1),
                   "tb_dt_s": round(t_tb, 1)},
        "stages_ms": {kk: sum(v) / len(v) for kk, v in stages.items()},
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                     "traffic": None, "peak_kind": peak_kind, "algorithmic_bytes": alg},
        "e2e": {"value": in_rows / e2e_s, "unit": "rows/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms": 1e3 * e2e_s},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, inst.config)
    print(json.dumps(line), flush=True)


def _pinned_copy(gpu, x):
    y = gpu.pinned_empty(x.shape, x.dtype)
    y[...] = x
    return y


def cpu_baseline(args, cfg):
    """The oracle merge (oracle/merge.hpp, one thread) on a bounded instance of
    the same distribution / dimension / k (the full config's inputs would take
    minutes in its std::set / sorted-index restatement)."""
    import oracle
    from paper_1902_07554_b200 import host
    inst = host.make_instance(args.config, n=args.cpu_n, k=args.k)
    lab = oracle.assign_kdtree(inst.points, inst.sample_ids, inst.sample_labels)
    P = host.attach_partials(inst, lab)
    fb = oracle.find_border(inst.points, lab, P)
    flags, vids = ((fb["border"], fb["vertices_border"]) if args.border == "bfs"
                   else (fb["positive"], fb["vertices_positive"]))
    tb = host.triangulate(inst.points, vids, 1)
    t = time.perf_counter()
    oracle.merge(P, flags, tb, lab)
    dt = time.perf_counter() - t
    rows = P.S + tb.verts.shape[1]
    return {"value": rows / dt, "unit": "rows/s", "cores": 1, "kind": "port",
            "sample": f"oracle merge on {inst.n} points of the same config ({rows} rows, {dt:.2f}s)"}


if __name__ == "__main__":
    main()
