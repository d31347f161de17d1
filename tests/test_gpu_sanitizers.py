"""compute-sanitizer over small launches of the hand-written kernels
(SURVEY §5): memcheck (out-of-bounds / misaligned accesses, leaks of device
errors), racecheck (shared-memory hazards, incl. the mbarrier / TMA / TMEM
pipelines of the tcgen05 GEMMs), synccheck (barrier misuse).  The kernels:
k_gemm_pair (2 digits and the 1-digit double-buffered mode), k_gemm_tc
(single-CTA, L = 4 and 2, the fused-check epilogue with its cross-CTA
counters, the scatter epilogue of the fused exchange), k_disentangle /
k_disentangle3x4, k_pinner and k_pinner_stream, the direct and Toeplitz
convolutions.  Pass = every case's oracle comparison holds under the tool
and the tool reports 0 errors."""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = "/usr/local/cuda/bin/compute-sanitizer"
CASES = ["pair", "pair1", "tc", "tc_check", "scatter", "check", "pinner", "conv"]


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "9",
           sys.executable, os.path.join(ROOT, "tests", "_sanitize_driver.py"), *CASES]
    if tool == "racecheck":
        cmd[3:3] = ["--racecheck-report", "hazard"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1800)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-5000:]
    for c in CASES:
        assert f"case {c} ok" in out, out[-3000:]
    m = re.search(r"ERROR SUMMARY: (\d+) error", out)
    assert m and int(m.group(1)) == 0, out[-5000:]
