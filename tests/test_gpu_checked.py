"""The bounds-checked build (libsfft_b200_checked.so, -DSFFT_CHECKED: device
asserts on the gather indices, shared-memory rows, DSMEM slots, table columns
and row indices of the hot kernels) over every kernel family at small shapes
(tests/sanitize_driver.py) -- the stand-in for compute-sanitizer memcheck,
which is closed on this GPU pool.  A failed check traps the launch."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(os.path.dirname(HERE), "paper_2012_08238_b200", "libsfft_b200_checked.so")


def test_checked_build_clean():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(LIB):
        pytest.skip("checked build not present (build() makes it)")
    env = dict(os.environ, SFFT_LIB_PATH=LIB)
    r = subprocess.run([sys.executable, os.path.join(HERE, "sanitize_driver.py")], env=env,
                       capture_output=True, text=True, timeout=1800)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "SFFT_DASSERT" not in out, out[-4000:]
    assert out.count("sanitize:") >= 10, out[-2000:]
