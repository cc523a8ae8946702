"""GPU: the C++ drop-in façade (include/vmonarch_b200.hpp) against the unmodified reference
operator on the same vmonarch::Mat<float> inputs (oracle/dropin_test.cpp, built by
oracle/Makefile from the reference's own headers and sources into oracle/_ref/).  Checks
outputs and MonarchFactors to <= 1e-4 and that both raise the same exception classes."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "dropin_test")


def test_cpp_dropin_facade_matches_reference(cuda):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_test not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK: 0 failure(s)" in r.stdout
    assert r.stdout.count("[PASS]") >= 25
