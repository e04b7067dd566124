"""The reference's OWN acceptance suite (proj/tests/acceptance.cpp, eight
SPEC criteria), compiled unmodified against this repository's drop-in
headers and linked to libcsaidx.so (oracle/Makefile `acceptance`): every
driver / score / top-k call it makes runs on the B200. Built where
/root/reference exists; the binary travels to the GPU box in oracle/_ref."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "acceptance_b200")


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
