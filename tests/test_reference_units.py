"""The reference's own doctest unit tests (proj/tests/test_*.cpp, unmodified,
compiled by path against oracle/shim's doctest/Boost stand-ins and the
F4-patched sequential_dt.cpp). 30 of 32 pass; the two cospherical tie-break
cases fail by construction in the reference (its tie rule makes the
tie-broken validator reject every triangulation of a cocircular square), as
documented in DESIGN.md."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "ref_unit_tests")

KNOWN_REFERENCE_FAILURES = {
    "cocircular square resolves deterministically via the tie-break",
    "3d cospherical points are tie-broken consistently",
}


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref not built (reference tree absent)")
def test_reference_unit_tests():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    passed = [l[7:] for l in r.stdout.splitlines() if l.startswith("[PASS] ")]
    failed = [l[7:] for l in r.stdout.splitlines() if l.startswith("[FAIL] ")]
    assert len(passed) + len(failed) == 32
    assert set(failed) == KNOWN_REFERENCE_FAILURES, failed
