"""compute-sanitizer memcheck / racecheck / synccheck over every kernel family
at small shapes (tests/sanitize_driver.py).  Opt-in (minutes per tool):
SFFT_SANITIZE=1 python -m pytest tests/test_gpu_sanitize.py -m gpu.  The
committed logs are under profiles/ (r2_sanitize_*.txt)."""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
CS = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.skipif(os.environ.get("SFFT_SANITIZE") != "1", reason="opt-in (SFFT_SANITIZE=1)")
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    if not os.path.exists(CS):
        pytest.skip("compute-sanitizer not installed")
    r = subprocess.run([CS, "--tool", tool, "--error-exitcode", "7", sys.executable,
                        os.path.join(HERE, "sanitize_driver.py")],
                       capture_output=True, text=True, timeout=3600)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
