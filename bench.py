#!/usr/bin/env python3
"""Benchmark of the sample-based divide step's hot path on B200 (sm_100a).

One step = assign_points over all n points (nearest-sample labels + the
Partitioning.parts bucketing) followed by find_border over all k partial DTs
(owner grid, full-scan positive flags, border-vertex compaction) — the two
stages of BASELINE.json's north_star, inputs resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

N>1 (torchrun): one process per GPU; each rank owns an independent instance
of the config (seed derived from the rank) — weak scaling, no data-path
collective; rank 0 prints the max-over-ranks line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "input points partitioned/s and simplices border-tested/s on 1 B200; % HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=None, help="override n (test-scale runs)")
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--policy", default="grid")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-row-order", action="store_true", help="skip the slot-row-order leg")
    ap.add_argument("--ref-budget-s", type=float, default=180.0,
                    help="--impl reference: wall budget for the timed full CPU steps (at least 3 run)")
    ap.add_argument("--no-parity", action="store_true", help="skip the full-size parity leg (and the CPU baseline)")
    ap.add_argument("--profile", action="store_true", help="single short run for ncu (no baseline/e2e)")
    ap.add_argument("--no-graph", action="store_true",
                    help="time launched steps only (default: the headline times the step replayed as one CUDA graph)")
    return ap.parse_args()


def h2d_floor_ms(nbytes: int) -> float:
    """Time of one plain page-locked host-to-device copy of nbytes (the PCIe
    floor of the e2e step), CUDA events, best of 3."""
    import torch
    src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    best = float("inf")
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    del src, dst
    return best


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
def algorithmic_bytes(dim, n, S, cells, n_vb):
    b_assign = n * (8 * dim + 4)
    b_border = S * (4 * (dim + 1) + 1) + n * (8 * dim + 1) + cells * 2 + n_vb * 4
    return b_assign, b_border


def dropin_leg(exe, inst, part, steps):
    """e2e through the C++ drop-in headers (the reference-facing C++ API):
    the instance goes to a file, dropin_example times `steps` full steps."""
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        src = os.path.join(td, "instance.bin")
        with open(src, "wb") as f:
            f.write(np.array([inst.dim], np.uint32).tobytes() + np.array([inst.n], np.uint64).tobytes()
                    + np.array([len(inst.sample_ids), part.k], np.uint32).tobytes()
                    + np.array([part.S], np.uint64).tobytes())
            for a in (inst.points, inst.sample_ids, inst.sample_labels, part.offsets, part.verts, part.nbrs,
                      part.parity):
                f.write(np.ascontiguousarray(a).tobytes())
        try:
            r = subprocess.run([exe, src, os.path.join(td, "out.bin"), "--bench", str(steps)], capture_output=True,
                               text=True, timeout=600)
        except subprocess.TimeoutExpired:
            return {"error": "timeout"}
    if r.returncode != 0:
        return {"error": r.stderr.strip()[-300:]}
    d = json.loads(r.stdout.strip().splitlines()[-1])
    d.update(value=inst.n / (d["ms_per_step"] * 1e-3), unit="points/s",
             path="sbdt::assign_points + sbdt::build_grid_index + sbdt::find_border(BorderOptions{no BFS, "
                  "points resident}) on the reference's PointSet / Triangulation<D>, TaskPool(all threads), "
                  "host buffers (tests/cpp/dropin_example.cpp --bench)")
    return d


def ceilings(ctx):
    """Binding ceilings measured on this device (diagnostic C-ABI microbenchmarks):
    the DFMA issue peak and random 8-byte gathers from an L2-sized table (the
    prefilter's 80 MB packed coordinates) and from an HBM-sized one (2 GB,
    the exact stage's binary64 coordinates by PointId, ~L2-missing). The border
    kernels are gather-, latency- and issue-bound rather than bandwidth-bound;
    these are the ceilings their per-kernel fractions are read against
    (profiles/README.md)."""
    try:
        dfma = ctx.microbench("dfma")
        g80 = ctx.microbench("gather", 80 << 20)
        g2g = ctx.microbench("gather", 2 << 30)
    except Exception as e:  # diagnostic only
        return {"error": str(e)}
    return {"dfma_tflops": round(dfma / 1e12, 2), "gather8_l2_gps": round(g80 / 1e9, 1),
            "gather8_hbm_gps": round(g2g / 1e9, 1),
            "issue_peak_warp_inst_per_s": None,
            "note": "gathers/s of independent random 8-byte loads (4 in flight per thread, 148x16 CTAs of 256); "
                    "DFMA: 8 independent chains per thread"}


def config_dict(inst, policy, world, cells):
    """The `config` of both arms (identical keys and values)."""
    part = inst.partials
    return {"workload": inst.config["name"], "n": inst.n, "dim": inst.dim, "k": inst.config["k"],
            "m": len(inst.sample_ids), "S": part.S, "policy": f"{policy}(c_G=1)", "cells": cells,
            "l2": "inputs > L2 (coords %d MB, simplices %d MB); the GPU arm also writes a 256 MB buffer (> L2) "
                  "between steps" % (inst.points.nbytes >> 20, (part.verts.nbytes + part.nbrs.nbytes) >> 20),
            "row_order": "slot (construction order)" if os.environ.get("SBDT_HOST_ROW_ORDER") == "slot"
                         else "morton (the host DT builder's compacted row order)",
            "parallelism": f"{world} independent instance(s), one per rank"}


def single_core(inst, labels, policy, budget_s=8.0):
    """One host core (TaskPool(1), the reference's determinism baseline,
    task_pool.hpp:20-21) on a bounded sample: the first points and the first
    part, on the reference's compiled primitives (oracle/_ref) when built."""
    import oracle
    n, k = inst.n, inst.config["k"]
    n_s = min(n, 200_000)
    r = oracle.ref_time_step(inst.points, inst.sample_ids, inst.sample_labels, labels, inst.partials, policy,
                             threads=1, n_assign=n_s, parts=(0, 1))
    kind = "reference"
    if r is None:  # no oracle/_ref: the restatement on one thread
        import time as _t
        t0 = _t.perf_counter()
        lab = np.empty(n_s, np.uint32)
        oracle.assign_kdtree(inst.points[:n_s], inst.sample_ids, inst.sample_labels, 1)
        ta = _t.perf_counter() - t0
        o = oracle.find_border(inst.points, labels, inst.partials, policy, threads=1, parts=(0, 1))
        r, kind = {"times": (ta, o["times"][0], o["times"][1])}, "port"
    S1 = int(inst.partials.offsets[1])
    return {"cores": 1, "kind": kind, "assign_points_per_s": n_s / r["times"][0],
            "border_simplices_per_s": S1 / max(r["times"][2], 1e-9),
            "sample": f"{n_s} points assigned ({r['times'][0]:.2f}s), part 0 = {S1} simplices border-tested "
                      f"({r['times'][2]:.2f}s; its index build {r['times'][1]:.2f}s excluded)",
            "est_step_s": n * r["times"][0] / n_s + inst.partials.S * r["times"][2] / max(S1, 1)}


def parity_leg(inst, policy, threads, g):
    """Full-size parity of this run's GPU outputs against the CPU oracle on
    all host threads (oracle/parity.py), and the oracle's own measured times:
    the CPU path over ALL n points and ALL k partials (not a sample)."""
    from oracle import parity
    res, _ = parity.check_labels(inst.points, inst.sample_ids, inst.sample_labels, inst.config["k"], g["labels"],
                                 g["parts_offsets"], g["parts_ids"], threads)
    res.update(parity.check_border(inst.points, g["labels"], inst.partials, g["positive"], g["border"],
                                   g["positive_vertex_ids"], g["border_vertex_ids"], policy, threads))
    res["all_equal"] = parity.all_equal(res)
    res["checked"] = ("labels (all n), Partitioning.parts, positive + BFS border flags (all S rows), both vertex "
                      "sets vs the CPU oracle, bit for bit")
    return res


def cpu_baseline_from(par, inst, threads, one_core):
    import oracle
    t_step = par["assign_s"] + par["border_s"]
    return {"value": inst.n / t_step, "unit": "points/s", "cores": threads, "kind": "port",
            "cpu_model": oracle.cpu_model(),
            "sample": (f"full step measured, not extrapolated: all {inst.n} points assigned (kd-tree, "
                       f"{par['assign_s']:.2f}s) + all {inst.partials.S} simplex rows of the {inst.config['k']} "
                       f"partials border-tested (full scan + BFS, {par['border_s']:.2f}s; per-part GridIndex "
                       f"build {par['index_build_s']:.2f}s excluded, it is an input of find_border)"),
            "assign_points_per_s": inst.n / par["assign_s"],
            "border_simplices_per_s": inst.partials.S / par["border_s"], "step_s": t_step,
            "single_core": one_core}


# ---------------------------------------------------------------------------
def run_reference(args):
    """--impl reference: the CPU path on all host threads, full steps (all n
    points, all k partials), measured. On the reference's own compiled
    primitives (geometry.cpp) and TaskPool (oracle/_ref, kind "reference")
    when built, else the restatement (kind "port"); the reference ships no
    hot-path code of its own."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1902_07554_b200 import host
    import oracle
    threads = os.cpu_count() or 1
    inst = host.make_instance(args.config, n=args.n, k=args.k)
    labels = oracle.assign_kdtree(inst.points, inst.sample_ids, inst.sample_labels, threads)
    host.attach_partials(inst, labels, threads=threads)
    cells = int(np.prod(oracle.grid_params(inst.points, 1.0)[3]))
    kind = "reference" if oracle.ref_lib() is not None else "port"

    def step():
        if kind == "reference":
            r = oracle.ref_time_step(inst.points, inst.sample_ids, inst.sample_labels, labels, inst.partials,
                                     args.policy, threads=threads)
            return r["times"]
        t0 = time.perf_counter()
        oracle.assign_kdtree(inst.points, inst.sample_ids, inst.sample_labels, threads)
        ta = time.perf_counter() - t0
        o = oracle.find_border(inst.points, labels, inst.partials, args.policy, threads=threads)
        return (ta, o["times"][0], o["times"][1])

    # full steps within a wall budget: one warm-up, then up to --steps timed
    # steps (at least 3) while the budget lasts
    t_begin = time.perf_counter()
    step()
    steps, ts = [], []
    while len(steps) < max(1, args.steps):
        ts.append(step())
        steps.append(ts[-1][0] + ts[-1][2])
        if len(steps) >= 3 and time.perf_counter() - t_begin > args.ref_budget_s:
            break
    t = statistics.median(steps)
    v = inst.n / t
    ta = statistics.median(x[0] for x in ts)
    tb = statistics.median(x[2] for x in ts)
    one = single_core(inst, labels, args.policy)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "points/s", "n_gpus": args.gpus,
            "steps": len(steps), "steps_requested": args.steps, "warmup": 1, "ms_per_step": 1e3 * t,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE.json config)",
            "config": config_dict(inst, args.policy, args.gpus, cells),
            "cpu_baseline": {"value": v, "unit": "points/s", "cores": threads, "kind": kind,
                             "cpu_model": oracle.cpu_model(),
                             "sample": (f"full steps, measured: all {inst.n} points assigned (kd-tree, median "
                                        f"{ta:.2f}s) + all {inst.partials.S} simplex rows border-tested (median "
                                        f"{tb:.2f}s; per-part GridIndex build excluded), {len(steps)} timed steps "
                                        f"after 1 warm-up" + (", on the reference's geometry.cpp + TaskPool("
                                        f"{threads})" if kind == "reference" else ", oracle restatement")),
                             "assign_points_per_s": inst.n / ta, "border_simplices_per_s": inst.partials.S / tb,
                             "single_core": one},
            "stage_rates": {"assign_points_per_s": inst.n / ta, "border_simplices_per_s": inst.partials.S / tb},
            "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    from paper_1902_07554_b200 import gpu, host
    from paper_1902_07554_b200 import dist as sdist

    rank, local, world = sdist.world()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    threads = max(1, (os.cpu_count() or 1) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world))))
    seed = sdist.rank_seed(host.CONFIGS[args.config]["seed"], rank, world)  # independent instance per rank
    t_setup = time.time()
    inst = host.make_instance(args.config, n=args.n, k=args.k, seed=seed)
    dim, n, k, m = inst.dim, inst.n, inst.config["k"], len(inst.sample_ids)
    ctx = gpu.Context(local)
    stream = torch.cuda.Stream(dev)  # dedicated stream: events and kernels on the same queue
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)

    # ---- device-resident inputs and outputs
    d_xyz = torch.from_numpy(np.ascontiguousarray(inst.points)).to(dev)
    d_sid = torch.from_numpy(inst.sample_ids.view(np.int32)).to(dev)
    d_slab = torch.from_numpy(inst.sample_labels.view(np.int32)).to(dev)
    d_lab = torch.empty(n, dtype=torch.int32, device=dev)
    d_poff = torch.empty(k + 1, dtype=torch.int64, device=dev)
    d_pids = torch.empty(n, dtype=torch.int32, device=dev)
    d_bbox = torch.empty(2 * dim, dtype=torch.int64, device=dev)
    P = lambda t: t.data_ptr()  # noqa: E731

    def assign():
        ctx.assign_points_dev(dim, P(d_xyz), n, P(d_sid), P(d_slab), m, k, P(d_lab), P(d_poff), P(d_pids), P(d_bbox))

    assign()
    torch.cuda.synchronize()
    labels = d_lab.cpu().numpy().view(np.uint32).copy()
    host.attach_partials(inst, labels, threads=threads)
    part = inst.partials
    S = part.S
    setup_s = time.time() - t_setup

    d_off = torch.from_numpy(part.offsets.view(np.int64)).to(dev)
    d_verts = torch.from_numpy(part.verts.view(np.int32)).to(dev)
    d_nbrs = torch.from_numpy(part.nbrs.view(np.int32)).to(dev)
    d_par = torch.from_numpy(part.parity).to(dev)
    d_pos = torch.empty(S, dtype=torch.uint8, device=dev)
    d_bor = torch.empty(S, dtype=torch.uint8, device=dev)
    d_vf = torch.empty(n + 64, dtype=torch.uint8, device=dev)
    d_vids = torch.empty(n, dtype=torch.int32, device=dev)
    d_cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    d_bvf = torch.empty(n + 64, dtype=torch.uint8, device=dev)
    d_bvids = torch.empty(n, dtype=torch.int32, device=dev)
    d_bcnt = torch.zeros(1, dtype=torch.int64, device=dev)

    def border_args(bfs: bool, rows=None):
        a = gpu.BorderArgs()
        a.dim, a.d_xyz, a.n, a.d_labels, a.k = dim, P(d_xyz), n, P(d_lab), k
        r_off, r_verts, r_nbrs, r_par = rows or (d_off, d_verts, d_nbrs, d_par)
        a.d_offsets, a.d_verts, a.d_nbrs, a.d_parity, a.S = P(r_off), P(r_verts), P(r_nbrs), P(r_par), S
        a.policy, a.c_G, a.flags = gpu.POLICY[args.policy], 1.0, gpu.HULL_BFS if bfs else 0
        a.d_bbox_ordered = P(d_bbox)
        a.d_positive, a.d_border = P(d_pos), P(d_bor) if bfs else None
        a.d_vertex_flags, a.d_vertex_ids, a.d_vertex_count = P(d_vf), P(d_vids), P(d_cnt)
        if bfs:
            a.d_bfs_vertex_flags, a.d_bfs_vertex_ids, a.d_bfs_vertex_count = P(d_bvf), P(d_bvids), P(d_bcnt)
        return a

    args_full, args_bfs = border_args(False), border_args(True)

    def step(bfs=False):
        assign()
        ctx.find_border_dev(args_bfs if bfs else args_full)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def timed(nsteps, bfs=False):
        ctx.set_timing(True)
        ms, stages = [], {}
        l0 = ctx.launches
        for _ in range(nsteps):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            step(bfs)
            e.record(stream)
            e.synchronize()
            ms.append(s.elapsed_time(e))
            for name, t in ctx.stage_times():
                stages.setdefault(name, []).append(t)
        ctx.set_timing(False)
        return ms, {kk: sum(v) / len(v) for kk, v in stages.items()}, ctx.launches - l0

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    ctx.synchronize()  # surfaces device-side status (degenerate simplex, grid cap)

    # one step captured as a CUDA graph (every launch, memset and cross-stream
    # fork/join of assign_points_dev + find_border_dev), replayed per step
    graph_ms, gms = None, []
    if not args.no_graph and not args.profile:
        pos_ref, cnt_ref, lab_ref = d_pos.clone(), d_cnt.clone(), d_lab.clone()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            step()
        for it in range(max(args.warmup, 0) + args.steps):
            flush.zero_()
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_.record(stream)
            g.replay()
            e_.record(stream)
            e_.synchronize()
            if it >= max(args.warmup, 0):
                gms.append(s_.elapsed_time(e_))
        ctx.synchronize()
        # the replayed step computes exactly what the launched step did
        assert torch.equal(d_pos, pos_ref) and torch.equal(d_cnt, cnt_ref) and torch.equal(d_lab, lab_ref)
        graph_ms = sum(gms) / len(gms)
        del g, pos_ref, cnt_ref, lab_ref

    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_wall0 = time.perf_counter()
        ms, stages, launches = timed(args.steps)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
    if dist:
        dist.barrier()
    # device time, max over ranks: the step replayed as a CUDA graph (the
    # launched steps give the per-stage events and the launch count)
    total_ms = sdist.max_over_ranks(sum(gms) if gms else sum(ms), device=dev)
    ctx.synchronize()
    # pipeline census: one extra, untimed step with the counters on
    ctx.set_timing(False, census=True)
    step()
    ctx.synchronize()
    table_stats = ctx.table_stats()
    border_stats = ctx.border_stats()
    ctx.set_timing(False)

    n_vb = int(d_cnt.item())
    # SPEC find_border (hull-seeded BFS) variant, timed separately (K8 included),
    # after one untimed step (its workspaces are allocated there)
    step(bfs=True)
    torch.cuda.synchronize()
    ms_bfs, stages_bfs, _ = timed(max(1, min(args.steps, 5)), bfs=True)
    n_vb_bfs = int(d_bcnt.item())
    n_pos = int(d_pos.sum().item())

    # Row-order leg: the bench's partial DTs come from this repo's host builder,
    # which emits rows along a Morton curve. The same
    # step on the builder's slot order (the order of its construction, what a
    # caller with spatially unordered rows sees), launched, a few steps.
    row_order = None
    if rank == 0 and world == 1 and not args.profile and not args.no_row_order \
            and os.environ.get("SBDT_HOST_ROW_ORDER") != "slot":
        keep = args_full
        try:
            os.environ["SBDT_HOST_ROW_ORDER"] = "slot"
            try:
                part_s = host.build_partials(inst.points, labels, k, inst.config["seed"], threads)
            finally:
                del os.environ["SBDT_HOST_ROW_ORDER"]
            assert part_s.S == S and np.array_equal(part_s.offsets, part.offsets)
            rows_s = (d_off, torch.from_numpy(part_s.verts.view(np.int32)).to(dev),
                      torch.from_numpy(part_s.nbrs.view(np.int32)).to(dev), torch.from_numpy(part_s.parity).to(dev))
            args_full = border_args(False, rows_s)
            for _ in range(2):
                step()
            torch.cuda.synchronize()
            ms_s, stages_s, _ = timed(max(1, min(args.steps, 5)))
            ctx.synchronize()
            assert int(d_pos.sum().item()) == n_pos and int(d_cnt.item()) == n_vb  # the same border, other row ids
            row_order = {"bench": "morton", "morton_launched_ms": round(sum(ms) / len(ms), 4),
                         "slot_launched_ms": round(sum(ms_s) / len(ms_s), 4),
                         "slot_prefilter_ms": round(stages_s.get("border.prefilter", 0.0), 4),
                         "morton_prefilter_ms": round(stages.get("border.prefilter", 0.0), 4)}
            del rows_s, part_s
        except Exception as exc:  # a side leg: never takes the bench line down
            row_order = {"bench": "morton", "error": f"{type(exc).__name__}: {exc}"[:200]}
        finally:
            args_full = keep
        step()  # the device outputs of the bench's own rows again (parity leg below)
        torch.cuda.synchronize()
    # this run's device outputs, for the full-size parity leg
    u32 = lambda t: t.cpu().numpy().view(np.uint32)  # noqa: E731
    g_out = {"labels": u32(d_lab), "parts_offsets": d_poff.cpu().numpy().view(np.uint64),
             "parts_ids": u32(d_pids), "positive": d_pos.cpu().numpy(), "border": d_bor.cpu().numpy(),
             "positive_vertex_ids": u32(d_vids[:n_vb]), "border_vertex_ids": u32(d_bvids[:n_vb_bfs])}

    import oracle  # checker only: grid cell count for the byte model
    lo, hi, edge, dims = oracle.grid_params(inst.points, 1.0)
    cells = int(np.prod(dims))
    b_assign, b_border = algorithmic_bytes(dim, n, S, cells, n_vb)
    peak, peak_kind = peaks()

    # DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) from
    # the committed ncu --set full capture of the same command (config 2)
    traffic_by_stage, inst_by_stage = {}, {}
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
    if os.path.exists(tpath) and args.config == 2 and args.n is None and args.policy == "grid":
        with open(tpath) as f:
            tj = json.load(f)
            traffic_by_stage, inst_by_stage = tj.get("stages", {}), tj.get("inst", {})
    issue_peak = torch.cuda.get_device_properties(dev).multi_processor_count * 4 * 1965e6  # warp inst/s

    def roof(bytes_, ms_, stage=None):
        a = bytes_ / (ms_ * 1e-3) / 1e9
        t = traffic_by_stage.get(stage)
        r = {"bound": "hbm", "achieved": round(a, 1), "peak": peak, "unit": "GB/s", "frac": round(a / peak, 4),
             "traffic": int(t) if t else None, "algorithmic_bytes": int(bytes_), "ms": round(ms_, 4),
             "peak_kind": peak_kind}
        ins = inst_by_stage.get(stage)
        if ins:
            # the binding ceiling of these gather/latency-bound kernels: the
            # issue rate (one warp instruction per SMSP per clock; ncu's
            # instruction count of the same kernel per launch)
            r["issue_frac"] = round(ins / (ms_ * 1e-3) / issue_peak, 4)
        return r

    # stages timed on the side stream overlap the launch stream's kernels
    # (find_border runs the hull rows' halfspace kernel next to exact + wide):
    # they count neither in the serial stage sums nor as the dominant kernel
    overlapped = {"border.infinite", "border.wide"} if args.policy in ("grid", "exact") and S > 0 else set()
    t_assign = sum(v for kk, v in stages.items() if kk.startswith("assign."))
    t_border = sum(v for kk, v in stages.items() if kk.startswith("border.") and kk not in overlapped)
    n_cand = int(border_stats.get("exact_stage_rows", 0))   # binary64 exact stage
    n_scan = int(border_stats.get("scan32_rows", 0))        # binary32 cell scan
    n_wide = int(border_stats.get("wide_rows", 0))          # pyramid descents routed by the prefilter
    # algorithmic bytes per launch (SURVEY.md 8d per unit x the units of one launch):
    kernel_bytes = {
        "assign.points": n * (8 * dim + 4),
        "border.finite": S * (4 * (dim + 1) + 1) + n * (8 * dim + 4 + 1) + cells * 2,
        # prefilter: vertex ids + flag per row, the 8-byte packed coordinate of
        # every point once, one 8-byte field word per cell once, and its queue
        # records (binary32 scan {row, U, Rp, reach}, wide {row, ids})
        "border.prefilter": S * (4 * (dim + 1) + 1) + n * 8 + cells * 8 + n_scan * 4 * (dim + 3)
        + n_wide * 4 * (dim + 2),
        # binary32 scan: its queue record and flag per row, field words once
        "border.scan32": n_scan * (4 * (dim + 3) + 1) + cells * 8,
        # binary64 exact stage: queue entry + ids + flag per row, coordinates once
        "border.exact": n_cand * (8 + 4 * (dim + 1) + 1) + n * 8 * dim + cells * 8,
        # owner grid: coordinates + labels in, packed coordinates out; owner
        # codes (2 B) and field words (8 B) per cell
        "border.grid": n * (8 * dim + 4 + 8) + cells * 10,
        "assign.bucket": n * 12,
        "border.compact": n + n_vb * 4,
    }
    dominant = max(((kk, v) for kk, v in stages.items() if kk not in overlapped), key=lambda kv: kv[1])[0]
    per_kernel = {kk: roof(kernel_bytes[kk], v, kk) for kk, v in stages.items() if kk in kernel_bytes}
    roofline = per_kernel.get(dominant) or roof(b_border, t_border)
    roofline = dict(roofline, kernel=dominant)

    value = sdist.aggregate_throughput(n, world, total_ms / args.steps * 1e-3)
    clocks = clk.summary()
    ceil = ceilings(ctx) if rank == 0 and not args.profile else None
    if ceil and "error" not in ceil:
        sm = torch.cuda.get_device_properties(dev).multi_processor_count
        ceil["issue_peak_warp_inst_per_s"] = sm * 4 * (clocks.get("sm_mhz") or 1965.0) * 1e6

    # ---- end to end through the host-buffer C ABI (pinned buffers; H2D+D2H inside)
    e2e = None
    if not args.no_e2e and not args.profile:
        def pinned(a):
            v = gpu.pinned_empty(a.shape, a.dtype)
            v[...] = a
            return v
        h_pts, h_sid, h_slab = pinned(np.ascontiguousarray(inst.points)), pinned(inst.sample_ids), pinned(inst.sample_labels)
        from paper_1902_07554_b200.host import Partials
        h_part = Partials(pinned(part.offsets), pinned(part.verts), pinned(part.nbrs), pinned(part.parity))
        ectx = gpu.Context(local)
        pol = gpu.IntersectionPolicy(args.policy, 1.0)
        # page-locked output buffers, allocated once (a serving loop reuses them)
        out_a = gpu.Partitioning(gpu.pinned_empty(n, np.uint32), gpu.pinned_empty(k + 1, np.uint64),
                                 gpu.pinned_empty(n, np.uint32), h_sid, h_slab, gpu.pinned_empty(2 * dim, np.float64))
        out_b = gpu.BorderSet(gpu.pinned_empty(S, np.uint8), None, None, gpu.pinned_empty(n, np.uint32))
        res = gpu.assign_points(h_pts, h_sid, h_slab, k, ctx=ectx, out=out_a)  # warm-up (allocations)
        gpu.find_border(h_pts, res.labels, h_part, pol, hull_bfs=False, ctx=ectx, out=out_b, resident=True)
        e2e_steps = max(1, min(args.steps, 3))
        t_calls = [0.0, 0.0]
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            ta = time.perf_counter()
            res = gpu.assign_points(h_pts, h_sid, h_slab, k, ctx=ectx, out=out_a)
            tb = time.perf_counter()
            # the points and labels of this step are still resident from assign_points
            bs = gpu.find_border(h_pts, res.labels, h_part, pol, hull_bfs=False, ctx=ectx, out=out_b, resident=True)
            t_calls[0] += tb - ta
            t_calls[1] += time.perf_counter() - tb
        t_e2e = (time.perf_counter() - t0) / e2e_steps
        assert np.array_equal(res.labels, labels)
        # find_border without the BFS reads only the last neighbour row (hull rows)
        # (the hull rows' neighbour is read in place from the page-locked
        # nbrs buffer: ~1% of S entries cross PCIe, counted as 4 B each)
        n_hull = int(np.count_nonzero(part.verts[dim] == 0xFFFFFFFF))
        # (parity crosses only for the exact policy, which orients in_sphere with it)
        h2d = (inst.points.nbytes + 8 * m + 8 * m * dim) + (part.offsets.nbytes + part.verts.nbytes + 4 * n_hull
                                                            + (part.parity.nbytes if args.policy == "exact" else 0))
        d2h = (4 * n + 8 * (k + 1) + 4 * n + 8 * dim) + (S + 8 + 4 * len(bs.positive_vertex_ids))
        e2e = {"value": world * n / t_e2e, "unit": "points/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": round(1e3 * t_e2e, 3),
               "call_ms": {"assign_points": round(1e3 * t_calls[0] / e2e_steps, 3),
                           "find_border": round(1e3 * t_calls[1] / e2e_steps, 3)},
               "h2d_floor_ms": round(h2d_floor_ms(h2d), 3),
               "path": "sbdt_gpu_assign_points + sbdt_gpu_find_border(RESIDENT_POINTS) (host buffers, pinned)"}
        ectx.close()

    # ---- the C++ drop-in path (include/sbdt/*.hpp on the reference's own
    # PointSet / Triangulation<D>, tests/cpp/dropin_example.cpp --bench):
    # assign_points + build_grid_index + find_border(no BFS, points resident)
    # on a TaskPool of all host threads, host buffers, wall clock per step
    dropin = None
    exe = os.path.join(ROOT, "paper_1902_07554_b200", "dropin_example")
    if rank == 0 and world == 1 and not args.no_e2e and not args.profile and os.path.exists(exe):
        dropin = dropin_leg(exe, inst, part, max(1, min(args.steps, 5)))

    cpu, par = None, None
    if rank == 0 and world == 1 and not args.no_parity and not args.profile:
        cores = os.cpu_count() or 1
        par = parity_leg(inst, args.policy, cores, g_out)
        if not args.no_cpu_baseline:
            cpu = cpu_baseline_from(par, inst, cores, single_core(inst, labels, args.policy))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json config)",
            "config": config_dict(inst, args.policy, world, cells),
            "parity": par,
            "stages_ms": {kk: round(v, 4) for kk, v in stages.items()},
            "overlapped_stages": sorted(overlapped),
            "launched_ms_per_step": round(sum(ms) / len(ms), 4),
            "timing": "CUDA graph replay of one step" if gms else "launched steps",
            "stage_rates": {"assign_points_per_s": n / (t_assign * 1e-3), "border_simplices_per_s": S / (t_border * 1e-3),
                            "assign_roofline": roof(b_assign, t_assign), "border_roofline": roof(b_border, t_border)},
            "roofline": roofline,
            "kernel_rooflines": per_kernel,
            "ceilings": ceil,
            "hull_bfs": {"ms_per_step": round(sum(ms_bfs) / len(ms_bfs), 4),
                         "stages_ms": {kk: round(v, 4) for kk, v in stages_bfs.items()},
                         "border_vertices": n_vb_bfs},
            "row_order": row_order,
            "border_vertices": n_vb, "positive_simplices": n_pos, "assign_table": table_stats, "border_pipeline": border_stats,
            "gpu_launches": int(launches), "gpu_launches_per_step": launches / args.steps,
            "clocks": clocks, "wall_timed_s": round(t_wall, 3), "setup_s": round(setup_s, 1),
            "e2e": e2e, "e2e_dropin": dropin, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
