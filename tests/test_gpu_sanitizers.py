"""compute-sanitizer over one small call of every device path (race and sync
detection for the mbarrier / TMA-ring / DSMEM / epoch-partial kernels).

`tools/sanitize_driver.py` runs kernels 3 (cluster ring), 5/6 (M = 2, 3..4 rings), 8 (all-SM
streaming: M = 1, MW = 2/4/8, fused segments, block-wise scaled LUTs and per-query scales), 9
(the persistent decode program, when built) and the generic canonical kernel, and itself exits
non-zero if any result misses the oracle bar.  Each tool must report "0 errors"."""

import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    for c in ("/usr/local/cuda/bin/compute-sanitizer", shutil.which("compute-sanitizer")):
        if c and os.path.exists(c):
            return c
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_reports_no_errors(tool):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "17", "--print-limit", "20",
           sys.executable, os.path.join(ROOT, "tools", "sanitize_driver.py")]
    if tool == "racecheck":
        cmd[3:3] = ["--racecheck-report", "all"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = res.stdout + res.stderr
    tail = "\n".join(out.splitlines()[-40:])
    if "closed on this pool" in out:
        # the GPU pool disables compute-sanitizer (it has left GPUs needing a reset); the
        # in-kernel guards (bounded spins that trap, shape checks before launch) and the
        # parity tests remain
        pytest.skip("compute-sanitizer is disabled on this GPU pool: " + out.strip().splitlines()[-1][:200])
    assert res.returncode == 0, tail
    assert "sanitize driver ok" in out, tail
    m = re.search(r"ERROR SUMMARY: (\d+) error", out)
    assert m is not None and int(m.group(1)) == 0, tail
    if tool == "racecheck":
        h = re.search(r"RACECHECK SUMMARY: (\d+) hazard", out)
        assert h is None or int(h.group(1)) == 0, tail
