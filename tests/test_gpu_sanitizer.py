"""compute-sanitizer over one small decode step of every kernel family (tools/sanitize_case.py): memcheck
(out-of-bounds / misaligned accesses), racecheck (shared-memory hazards, incl. the TMA / mbarrier staging and
the DSMEM merges), synccheck (barrier misuse) and initcheck (reads of uninitialised device memory).
Each must report 0 errors (race and failure detection)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_sanitizer_clean(tool):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    # device-side checks only: CUDA API errors are the library's own business (every launch / API failure is
    # returned as TLS_ERR_CUDA), and the runtime's internal lazy-loading probe (cuKernelGetFunction on first
    # launch) would be reported as one
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20", "--report-api-errors", "no"]
    r = subprocess.run(cmd + [sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py")], capture_output=True,
                       text=True, timeout=1500, cwd=ROOT)
    out = r.stdout + r.stderr
    if "compute-sanitizer is closed" in out:  # the GPU pool's wrapper refuses the tool (not this library's result)
        pytest.skip("compute-sanitizer is disabled on this GPU pool: " + out.strip().splitlines()[-1][:200])
    assert r.returncode == 0 and "sanitize cases done" in out, out[-4000:]
    summary = "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" if tool == "racecheck" else \
        "ERROR SUMMARY: 0 errors"
    assert summary in out, out[-4000:]
