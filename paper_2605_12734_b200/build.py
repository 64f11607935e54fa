"""Builds libjacobi3d.so in-tree with nvcc for sm_100a (no JIT cache, so the .so
travels to the GPU box with the repo snapshot).

Flags: -gencode arch=compute_100a,code=sm_100a, -fmad=false (north star: fixed
summation order, no contraction), -lineinfo (ncu source page), -O3.

``build(checked=True)`` builds libjacobi3d_checked.so with -DJAC_CHECKED: every kernel
store range- and alignment-checked, TMA coordinates asserted (device.hpp CheckArgs) --
the test-only substitute for compute-sanitizer, which is closed on this GPU pool.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libjacobi3d.so")
LIB_CHECKED = os.path.join(PKG, "libjacobi3d_checked.so")
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


def _lib(checked: bool) -> str:
    return LIB_CHECKED if checked else LIB


def _flags(checked: bool):
    return NVCC_FLAGS + (["-DJAC_CHECKED"] if checked else [])


def _digest(checked: bool = False) -> str:
    import hashlib
    h = hashlib.sha256(" ".join(_flags(checked)).encode())
    for f in _inputs():
        with open(f, "rb") as fh:
            h.update(os.path.basename(f).encode() + b"\0" + fh.read())
    return h.hexdigest()


def needs_build(checked: bool = False) -> bool:
    """Content-based: a copied tree (new mtimes, e.g. the gpurun snapshot) reuses a
    .so built from the same sources; without a stamp, fall back to mtimes."""
    lib = _lib(checked)
    stamp = lib + ".stamp"  # sha256 of the inputs + flags the .so was built from
    if not os.path.exists(lib):
        return True
    if os.path.exists(stamp):
        with open(stamp) as fh:
            return fh.read().strip() != _digest(checked)
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(f) > t for f in _inputs())


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    lib = _lib(checked)
    if not force and not needs_build(checked):
        return lib
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [nvcc, *_flags(checked), "-I", os.path.join(ROOT, "include"), "-o", tmp,
           *[os.path.join(CSRC, s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    digest = _digest(checked)
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    stamp = lib + ".stamp"
    with open(stamp + f".tmp{os.getpid()}", "w") as fh:
        fh.write(digest + "\n")
    os.replace(stamp + f".tmp{os.getpid()}", stamp)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv))
