"""compute-sanitizer over the sampling kernels on a small config:
memcheck (out-of-bounds / misaligned accesses), racecheck (shared-memory
hazards in the warp-synchronous K2 and K1 group kernels), synccheck (illegal
__syncwarp / barrier use) and initcheck (reads of uninitialised device memory),
each reporting zero errors while the outputs still equal the oracle's
(scripts/sanitize_case.py covers K0, K1 serial / group variants, both K2
kernels, the offset scan, K3 and the standalone gather)."""
import os
import shutil
import subprocess
import sys

import pytest

from tests.helpers import ROOT

pytestmark = pytest.mark.gpu

SANITIZER = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


def _sanitizer_usable() -> str | None:
    """None when compute-sanitizer can run here, else why not. The runs are
    opt-in (HGS_SANITIZE=1): the shared GPU pool closed the tool (a stub that
    prints a notice instead of running), so the suite must not depend on it;
    the logs of the last permitted runs are under profiles/r2_sanitizer/."""
    if not os.environ.get("HGS_SANITIZE"):
        return "compute-sanitizer runs are opt-in (HGS_SANITIZE=1); logs in profiles/r2_sanitizer/"
    try:
        res = subprocess.run([SANITIZER, "--version"], capture_output=True, text=True, timeout=60)
    except (OSError, subprocess.TimeoutExpired) as e:
        return f"compute-sanitizer not runnable: {e}"
    if "Compute Sanitizer" not in res.stdout + res.stderr:
        return "compute-sanitizer unavailable: " + (res.stdout + res.stderr).strip()[:200]
    return None


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_sanitizer_clean(tool):
    why = _sanitizer_usable()
    if why:
        pytest.skip(why)
    cmd = [SANITIZER, "--tool", tool, "--error-exitcode", "99", "--target-processes", "all", "--print-limit", "1000000"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    cmd += [sys.executable, os.path.join(ROOT, "scripts", "sanitize_case.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = res.stdout + res.stderr
    log = os.path.join(ROOT, "gpurun_out", f"sanitizer_{tool}.log")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    with open(log, "w") as f:
        f.write(out)
    assert "SANITIZE CASE OK" in out, out[-3000:]
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-3000:]
    assert "Potential" not in out and "hazard detected" not in out, out[:3000]
    assert res.returncode == 0, out[-3000:]
