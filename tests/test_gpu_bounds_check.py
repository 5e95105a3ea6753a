"""Every device path of tools/sanitize_driver.py against the bounds-checked debug build
(tools/check_build.sh, -DSHIFTADD_BOUNDS_CHECK): shared-memory accesses through the wrappers,
bulk-copy destinations, DSMEM stores and split-K partial-word stores trap on any address
outside the launch's dynamic shared memory / partial region.  This pool disables
compute-sanitizer (tests/test_gpu_sanitizers.py skips), so this is the memory-safety check
that runs; the driver also checks every result against the oracle."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2406_05981_b200", "libshiftadd_chk.so")


def test_bounds_checked_build_runs_every_path_clean():
    srcs = [os.path.join(ROOT, "paper_2406_05981_b200", "csrc", f)
            for f in os.listdir(os.path.join(ROOT, "paper_2406_05981_b200", "csrc"))]
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(f) for f in srcs):
        subprocess.run(["bash", os.path.join(ROOT, "tools", "check_build.sh")], check=True, timeout=900)
    env = dict(os.environ, SHIFTADD_LIB_PATH=LIB)
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_driver.py")], env=env,
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-3000:]
    assert "sanitize driver ok" in out
