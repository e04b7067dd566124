"""compute-sanitizer over the hand-written kernels:
memcheck (out-of-bounds / misaligned accesses), racecheck (shared-memory
hazards) and synccheck (barrier misuse) on small workloads that drive every
kernel family through the C-ABI (scripts/sanitize_case.py): the V4 step
(tcgen05 score + fused select), an exact-kernel key tiling (select + merge +
finalize), the select's sampled / heavy-tie / exact-fallback / large-take
paths, the persistent multi-row select, the two-level select and the sparse
attention kernel. Each run
must report zero errors / hazards."""
import os
import shutil
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SANITIZER = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(SANITIZER):
        pytest.fail("compute-sanitizer missing from the CUDA toolkit")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("case", ["smoke", "select", "persistent", "two_level", "attention", "attention_pair"])
def test_sanitizer_reports_no_hazards(tool, case):
    if case == "attention_pair" and tool == "racecheck":
        # the opt-in pair kernel hands the running max between its two
        # softmax teams with __syncwarp + one arrive per warp, which racecheck
        # does not model (per-lane arrivals here gave wrong results); memcheck
        # and synccheck run on it
        pytest.skip("racecheck does not model the warp-level max hand-off of the opt-in pair kernel")
    cmd = [SANITIZER, "--tool", tool, "--error-exitcode", "7", "--print-limit", "20", sys.executable,
           os.path.join(ROOT, "scripts", "sanitize_case.py"), case]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert f"cases ok: {case}" in out, out[-4000:]
    summary = "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" if tool == "racecheck" \
        else "ERROR SUMMARY: 0 errors"
    assert summary in out, out[-4000:]
