"""GPU: the C++ drop-in adapter (include/semwarm_b200.hpp) instantiated with the reference's
own semwarm:: types, compared result-for-result with the reference's IvfIndex and choose_arm
(tools/dropin_check.cpp, built against /root/reference headers into oracle/_ref/)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_check")


@pytest.mark.parametrize("dim,n", [(128, 800), (512, 1500), (64, 300)])
def test_cpp_dropin_matches_reference(dim, n):
    if not os.path.exists(BIN):
        pytest.skip("dropin_check not built (needs /root/reference at build time)")
    r = subprocess.run([BIN, str(dim), str(n)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "DROPIN PASS" in r.stdout, r.stdout + r.stderr
