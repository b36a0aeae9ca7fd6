"""The hull-row plane filter (csrc/common/plane_filter.hpp, used by
k_border_infinite) against the exact per-corner orient of predicates.hpp:
every box the filter decides (no / some / every corner strictly outside the
facet's plane, halfspace_box_overlap at geometry.cpp:329-345) must match the
exact classification, on random, on-plane and near-plane boxes over a wide
exponent range. Compiled with g++ (the same header the device includes)."""
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_plane_filter_matches_exact_orient(tmp_path):
    exe = tmp_path / "pfc"
    subprocess.run(["g++", "-O2", "-std=c++20", "-ffp-contract=off",
                    "-I" + os.path.join(ROOT, "paper_1902_07554_b200/csrc/common"), "-o", str(exe),
                    os.path.join(ROOT, "tests/cpp/plane_filter_check.cpp")], check=True)
    out = subprocess.run([str(exe), "200000"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["bad2"] == 0 and res["bad3"] == 0
    # the filter decides the large majority (the exact corners are the fallback)
    assert res["decided2"] > 0.7 * res["cases"] and res["decided3"] > 0.7 * res["cases"]
