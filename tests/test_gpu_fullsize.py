"""Full-size parity: every BASELINE.json config at its own n / k / sample
fraction (configs 1-5: 1M 2-D uniform, 10M 3-D uniform, 10M 3-D normal, 20M
3-D bubbles, 50M 2-D lines), GPU vs the CPU oracle on all host cores, bit for
bit (oracle/parity.py): labels of all n points, Partitioning.parts, the
full-scan positive flags and the SPEC BFS border flags of every simplex row of
all k partial DTs, and both border-vertex sets; the grid policy everywhere,
plus the exact policy on config 2. The pipeline census is recorded with each
run (dense-cell table builds on the clustered configs, escalation counters).

Ground truth: SPEC.md:342-350 (assign_points = brute-force nearest sample,
the kd-tree oracle equals it), :307-312 (parts), :418-433,451 (intersects),
:488-496 (find_border); the checker is pinned to the reference's compiled
primitives and golden vectors (tests/test_oracle.py)."""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import parity
from paper_1902_07554_b200 import gpu, host

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 8
_cache = {}


def _instance(cfg):
    if cfg not in _cache:
        _cache.clear()  # one full-size instance alive at a time (config 5: ~3.5 GB of host arrays)
        _cache[cfg] = host.make_instance(cfg)
    return _cache[cfg]


def _run(cfg, policy, ctx):
    inst = _instance(cfg)
    k = inst.config["k"]
    ctx.set_timing(False, census=True)
    try:
        part = gpu.assign_points(inst.points, inst.sample_ids, inst.sample_labels, k, ctx=ctx)
        table = ctx.table_stats()
        res, ref_labels = parity.check_labels(inst.points, inst.sample_ids, inst.sample_labels, k, part.labels,
                                              part.parts_offsets, part.parts_ids, THREADS)
        assert res["labels"], f"config {cfg}: labels differ: {res.get('labels_diff')}"
        assert res["parts"], f"config {cfg}: Partitioning.parts differ"
        if inst.partials is None:
            host.attach_partials(inst, part.labels, threads=THREADS)
        P = inst.partials
        bs = gpu.find_border(inst.points, part.labels, P, gpu.IntersectionPolicy(policy, 1.0), hull_bfs=True, ctx=ctx)
        census = ctx.border_stats()
    finally:
        ctx.set_timing(False)
    res.update(parity.check_border(inst.points, part.labels, P, bs.positive, bs.border, bs.positive_vertex_ids,
                                   bs.border_vertex_ids, policy, THREADS))
    rec = {"config": inst.config["name"], "policy": policy, "n": inst.n, "k": k, "m": len(inst.sample_ids),
           "S": P.S, "threads": THREADS, "parity": res, "assign_table": table,
           "census": {kk: census.get(kk) for kk in ("rows", "exact_stage_rows", "wide_rows", "orient_check_rows",
                                                    "orient_escalations", "in_sphere_escalations")}}
    print("FULLSIZE " + json.dumps(rec))
    for key in ("positive", "border", "positive_vertices", "border_vertices"):
        assert res[key], f"config {cfg} ({policy}): {key} differ: {res.get(key + '_diff')}"
    return rec


@pytest.mark.parametrize("cfg,policy", [(1, "grid"), (2, "grid"), (2, "exact"), (3, "grid"), (4, "grid"),
                                        (5, "grid")])
def test_fullsize(cfg, policy, ctx):
    _run(cfg, policy, ctx)
