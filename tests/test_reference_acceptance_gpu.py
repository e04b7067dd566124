"""The reference's OWN test suites, compiled unmodified against this
repository's drop-in headers and linked to libcsaidx.so (oracle/Makefile
`acceptance` and `unit`): the acceptance gate (proj/tests/acceptance.cpp,
eight SPEC criteria) and the 88 unit test cases (proj/tests/test_*.cpp; the
macros come from oracle/doctest_shim since doctest is not vendored). Every
driver / score / top-k call they make runs on the B200. Built where
/root/reference exists; the binaries travel to the GPU box in oracle/_ref."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

REF_BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
BIN = os.path.join(REF_BIN, "acceptance_b200")
UNIT = os.path.join(REF_BIN, "unit_b200")


def test_reference_acceptance_suite_passes_on_the_b200_library():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/acceptance_b200 not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=1200, cwd=os.path.dirname(BIN))
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "ACCEPTANCE: all 8 criteria passed" in out, out[-4000:]
    assert out.count("[PASS]") == 8, out[-4000:]


def test_reference_unit_tests_pass_on_the_b200_library():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(UNIT):
        pytest.skip("oracle/_ref/unit_b200 not built (needs /root/reference at build time)")
    r = subprocess.run([UNIT], capture_output=True, text=True, timeout=600, cwd=REF_BIN)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "test cases: 88 | 88 passed | 0 failed" in out, out[-4000:]
