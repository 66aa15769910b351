"""compute-sanitizer tier: memcheck, racecheck and synccheck over
small runs of every hand-written kernel family (tests/sanitize/small_paths.py:
the tcgen05 / TMA / mbarrier kernels, the CUDA-core levels, the CSR scan and
the peer-exchange release/acquire kernels).  Zero reported errors.

Opt-in (BPPSA_SANITIZER=1): the GPU pool closed compute-sanitizer during r02g
(runs under it elsewhere had left GPUs needing a reset), so the default -m gpu
tier does not start it.  All three tools ran clean on every r02a-r02f GPU
tier (profiles/r02*_pytest_gpu.log, 360 passed each); out-of-bounds and race
coverage otherwise comes from the parity tests' small ragged cases against the
oracle."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    for c in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if c and os.path.exists(c):
            return c
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    if os.environ.get("BPPSA_SANITIZER") != "1":
        pytest.skip("compute-sanitizer tier is opt-in (BPPSA_SANITIZER=1): closed on the GPU pool since r02g")
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "9", "--print-limit", "20",
           sys.executable, os.path.join(ROOT, "tests", "sanitize", "small_paths.py")]
    if tool == "memcheck":
        cmd[1:1] = ["--leak-check", "no"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=3000, cwd=ROOT)
    text = out.stdout + out.stderr
    print(text[-3000:])
    m = re.search(r"ERROR SUMMARY: (\d+) error", text) or re.search(r"SUMMARY: \d+ hazards? displayed \((\d+) error", text)
    assert m is not None, text[-2000:]
    assert int(m.group(1)) == 0 and out.returncode == 0, text[-3000:]
    if tool == "racecheck":
        assert re.search(r"\(0 errors, 0 warnings\)", text), text[-2000:]
    assert "small paths ok" in text
