"""bench.py's reference arm runs on CPU (no GPU needed) and prints the
contract's JSON line: one line, the same metric / unit / workload as the
product arm, a cpu_baseline describing the run and an e2e equal to the
line's own value (the driver computes the ratio itself)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--n", "20000",
                        "--k", "8", "--steps", "2", "--warmup", "0", "--ref-budget-s", "1"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["unit"] == "points/s" and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("cfg2") and d["config"]["n"] == 20000
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    # full steps measured (not extrapolated), a single-core figure and the CPU model
    assert d["steps"] >= 1 and "full steps, measured" in d["cpu_baseline"]["sample"]
    assert d["cpu_baseline"]["single_core"]["cores"] == 1 and d["cpu_baseline"]["cpu_model"]
    # the same config keys as the product arm (bench.config_dict)
    assert set(d["config"]) == {"workload", "n", "dim", "k", "m", "S", "policy", "cells", "l2", "row_order", "parallelism"}
