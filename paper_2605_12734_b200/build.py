"""Builds libjacobi3d.so in-tree with nvcc for sm_100a (no JIT cache, so the .so
travels to the GPU box with the repo snapshot).

Flags: -gencode arch=compute_100a,code=sm_100a, -fmad=false (north star: fixed
summation order, no contraction), -lineinfo (ncu source page), -O3.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libjacobi3d.so")
SOURCES = ["engine.cu", "kernels.cu", "microbench.cu", "plan.cpp"]
HEADERS = ["device.hpp", "kernels.hpp", "plan.hpp"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-Xcompiler", "-fvisibility=hidden",
]


def _inputs():
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "jacobi3d.h"))
    files.append(os.path.join(ROOT, "include", "jacobi3d_microbench.h"))
    files.append(os.path.abspath(__file__))
    return files


STAMP = LIB + ".stamp"  # sha256 of the inputs + flags the .so was built from


def _digest() -> str:
    import hashlib
    h = hashlib.sha256(" ".join(NVCC_FLAGS).encode())
    for f in _inputs():
        with open(f, "rb") as fh:
            h.update(os.path.basename(f).encode() + b"\0" + fh.read())
    return h.hexdigest()


def needs_build() -> bool:
    """Content-based: a copied tree (new mtimes, e.g. the gpurun snapshot) reuses a
    .so built from the same sources; without a stamp, fall back to mtimes."""
    if not os.path.exists(LIB):
        return True
    if os.path.exists(STAMP):
        with open(STAMP) as fh:
            return fh.read().strip() != _digest()
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _inputs())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", tmp,
           *[os.path.join(CSRC, s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    digest = _digest()
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    with open(STAMP + f".tmp{os.getpid()}", "w") as fh:
        fh.write(digest + "\n")
    os.replace(STAMP + f".tmp{os.getpid()}", STAMP)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
