"""The C++ drop-in: tests/cpp/dropin_test.cpp calls the reference (otpr) and
this library's C++ API (otprg, include/otprg.hpp) side by side and compares
the results field by field (assignment dense / points / rectangular, rounding,
errors, per-phase observer worksets + check_invariants, verify_feasibility,
OT plans, Sinkhorn).  The binary is built in the build container (it needs the
reference headers) and runs on the GPU box."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_bin", "dropin_test")


def test_cpp_dropin_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_bin/dropin_test not built (needs /root/reference headers)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
