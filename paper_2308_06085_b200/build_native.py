"""Build libhelmfree_b200.so in-tree with nvcc for sm_100a (no JIT cache).

Each translation unit is compiled to an object (in parallel, only when stale),
then the objects are linked into the shared library."""

from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

_HERE = os.path.dirname(os.path.abspath(__file__))
SOURCES = ["csrc/hf_kernels.cu", "csrc/hf_wide.cu", "csrc/hf_coarse_gmres.cu", "csrc/hf_runtime.cu"]
HEADERS = ["csrc/hf_device.cuh", "csrc/hf_kernels.cuh", "csrc/hf_stencil.cuh",
           "../include/helmfree_b200.h"]
OUT = os.path.join(_HERE, "_lib", "libhelmfree_b200.so")
OBJDIR = os.path.join(_HERE, "_lib", "obj")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
]


def _mtime(p: str) -> float:
    return os.path.getmtime(os.path.join(_HERE, p))


def _obj(src: str) -> str:
    return os.path.join(OBJDIR, os.path.basename(src).replace(".cu", ".o"))


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(_mtime(p) > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return OUT
    os.makedirs(OBJDIR, exist_ok=True)
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    hdr_t = max(_mtime(h) for h in HEADERS)

    def compile_one(src: str) -> None:
        obj = _obj(src)
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(_mtime(src), hdr_t):
            return
        cmd = [nvcc, *NVCC_FLAGS, "-c", "-o", obj, os.path.join(_HERE, src)]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True, cwd=_HERE)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as pool:
        list(pool.map(compile_one, SOURCES))
    cmd = [nvcc, "-Wno-deprecated-gpu-targets", "-shared", "-o", OUT + ".tmp", *[_obj(s) for s in SOURCES], "-lcusolver"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=_HERE)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
