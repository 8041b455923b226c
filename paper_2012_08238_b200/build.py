"""Build libsfft_b200.so in-tree with nvcc for sm_100a (no JIT cache, so the
library travels with the repo snapshot to the GPU box)."""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libsfft_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"]


def _stale(obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


CHECKED_OBJ = os.path.join(HERE, "_build_checked")
CHECKED_LIB = os.path.join(HERE, "libsfft_b200_checked.so")


def build(verbose: bool = False, jobs: int = 8, checked: bool = True) -> str:
    """The product library, and (checked=True) its bounds-checked twin
    libsfft_b200_checked.so (-DSFFT_CHECKED: device asserts on the hot
    kernels' indices; tests/test_gpu_checked.py runs it on small shapes)."""
    lib = _build(OBJ, LIB, [], verbose, jobs)
    if checked:
        _build(CHECKED_OBJ, CHECKED_LIB, ["-DSFFT_CHECKED"], verbose, jobs)
    return lib


def _build(OBJ: str, LIB: str, extra: list, verbose: bool, jobs: int) -> str:
    os.makedirs(OBJ, exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = sorted(glob.glob(os.path.join(CSRC, "*.cuh")))
    objs, todo = [], []
    for src in sources:
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if _stale(obj, [src] + headers):
            todo.append((src, obj))

    def compile_one(pair):
        src, obj = pair
        cmd = [NVCC, *FLAGS, *extra, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose and r.stderr.strip():
            print(r.stderr)
        return src

    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        for src in ex.map(compile_one, todo):
            if verbose:
                print("compiled", os.path.basename(src))
    if todo or _stale(LIB, objs):
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", LIB,
               "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
