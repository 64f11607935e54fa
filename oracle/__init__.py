"""CPU oracle for the overdecomposed Jacobi3D hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2605_12734_b200`` never imports it, and the two share no code.

``oracle_jacobi3d`` (C, ``jacobi3d_oracle.c``) is the plain undecomposed Jacobi
iteration of PAPER.md:281 (§5 jacobi2d, lifted to 3D per SURVEY.md §8(c) R1):
``B[p] = ((((((c + x-) + x+) + y-) + y+) + z-) + z+) * fl(1/7)`` on the padded
array, shell fixed.  ``oracle_np.jacobi3d_np`` is a second, independently written
numpy implementation used as pin P6.

Parity is pinned by tests/test_oracle_pins.py; no function here is "parity
unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "jacobi3d_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# -ffp-contract=off / -fno-fast-math: SURVEY.md §8(c.1) build flags (reading R5).
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-fopenmp"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (idempotent)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, dp = ctypes.c_int64, ctypes.POINTER(ctypes.c_double)
        L.oracle_jacobi3d.argtypes = [i64, i64, i64, dp, i64, dp]
        L.oracle_jacobi3d.restype = ctypes.c_int
        L.oracle_jacobi3d_timed.argtypes = [i64, i64, i64, dp, i64, dp, ctypes.POINTER(ctypes.c_double)]
        L.oracle_jacobi3d_timed.restype = ctypes.c_int
        L.oracle_jacobi3d_omp.argtypes = [i64, i64, i64, dp, i64, dp, ctypes.c_int]
        L.oracle_jacobi3d_omp.restype = ctypes.c_int
        L.oracle_jacobi3d_omp_timed.argtypes = [i64, i64, i64, dp, i64, dp, ctypes.c_int,
                                                 ctypes.POINTER(ctypes.c_double)]
        L.oracle_jacobi3d_omp_timed.restype = ctypes.c_int
        L.oracle_jacobi2d.argtypes = [i64, i64, dp, i64, dp]
        L.oracle_jacobi2d.restype = ctypes.c_int
        L.oracle_jacobi2d_omp.argtypes = [i64, i64, dp, i64, dp, ctypes.c_int]
        L.oracle_jacobi2d_omp.restype = ctypes.c_int
        L.oracle_jacobi2d_omp_timed.argtypes = [i64, i64, dp, i64, dp, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
        L.oracle_jacobi2d_omp_timed.restype = ctypes.c_int
        L.oracle_checksum.argtypes = [i64, i64, i64, dp]
        L.oracle_checksum.restype = ctypes.c_double
        L.oracle_bithash.argtypes = [i64, i64, i64, dp]
        L.oracle_bithash.restype = ctypes.c_uint64
        L.oracle_has_openmp.restype = ctypes.c_int
        _lib = L
    return _lib


def _dims(u: np.ndarray):
    if u.dtype != np.float64 or u.ndim != 3 or not u.flags.c_contiguous:
        raise ValueError("padded field must be a C-contiguous float64 array [nz+2, ny+2, nx+2]")
    nz2, ny2, nx2 = u.shape
    return nx2 - 2, ny2 - 2, nz2 - 2


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def jacobi3d(u0: np.ndarray, n: int) -> np.ndarray:
    """Padded field after ``n`` sweeps (single-threaded C oracle)."""
    nx, ny, nz = _dims(u0)
    out = np.empty_like(u0)
    rc = lib().oracle_jacobi3d(nx, ny, nz, _ptr(u0), int(n), _ptr(out))
    if rc != 0:
        raise RuntimeError(f"oracle_jacobi3d failed rc={rc}")
    return out


def jacobi3d_timed(u0: np.ndarray, n: int):
    """Single-threaded oracle (as ``jacobi3d``); returns (field, seconds of the
    iteration loop alone) -- the CPU baseline's mode (a)."""
    nx, ny, nz = _dims(u0)
    out = np.empty_like(u0)
    secs = ctypes.c_double()
    rc = lib().oracle_jacobi3d_timed(nx, ny, nz, _ptr(u0), int(n), _ptr(out), ctypes.byref(secs))
    if rc != 0:
        raise RuntimeError(f"oracle_jacobi3d_timed failed rc={rc}")
    return out, secs.value


def jacobi3d_omp(u0: np.ndarray, n: int, nthreads: int = 0):
    """OpenMP-over-z variant (pin P10). Returns (field, threads_used)."""
    nx, ny, nz = _dims(u0)
    out = np.empty_like(u0)
    rc = lib().oracle_jacobi3d_omp(nx, ny, nz, _ptr(u0), int(n), _ptr(out), int(nthreads))
    if rc < 1:
        raise RuntimeError(f"oracle_jacobi3d_omp failed rc={rc}")
    return out, rc


def jacobi3d_omp_timed(u0: np.ndarray, n: int, nthreads: int = 0):
    """Returns (field, threads_used, seconds of the iteration loop alone)."""
    nx, ny, nz = _dims(u0)
    out = np.empty_like(u0)
    secs = ctypes.c_double()
    rc = lib().oracle_jacobi3d_omp_timed(nx, ny, nz, _ptr(u0), int(n), _ptr(out), int(nthreads),
                                         ctypes.byref(secs))
    if rc < 1:
        raise RuntimeError(f"oracle_jacobi3d_omp_timed failed rc={rc}")
    return out, rc, secs.value


def _dims2(u: np.ndarray):
    if u.dtype != np.float64 or u.ndim != 2 or not u.flags.c_contiguous:
        raise ValueError("padded 2-D field must be a C-contiguous float64 array [ny+2, nx+2]")
    ny2, nx2 = u.shape
    return nx2 - 2, ny2 - 2


def jacobi2d(u0: np.ndarray, n: int) -> np.ndarray:
    """Jacobi2D (NEXT-1): padded 2-D field after ``n`` 5-point sweeps (serial C)."""
    nx, ny = _dims2(u0)
    out = np.empty_like(u0)
    rc = lib().oracle_jacobi2d(nx, ny, _ptr(u0), int(n), _ptr(out))
    if rc != 0:
        raise RuntimeError(f"oracle_jacobi2d failed rc={rc}")
    return out


def jacobi2d_omp(u0: np.ndarray, n: int, nthreads: int = 0):
    nx, ny = _dims2(u0)
    out = np.empty_like(u0)
    rc = lib().oracle_jacobi2d_omp(nx, ny, _ptr(u0), int(n), _ptr(out), int(nthreads))
    if rc < 1:
        raise RuntimeError(f"oracle_jacobi2d_omp failed rc={rc}")
    return out, rc


def jacobi2d_omp_timed(u0: np.ndarray, n: int, nthreads: int = 0):
    """Returns (field, threads_used, seconds of the iteration loop alone)."""
    nx, ny = _dims2(u0)
    out = np.empty_like(u0)
    secs = ctypes.c_double()
    rc = lib().oracle_jacobi2d_omp_timed(nx, ny, _ptr(u0), int(n), _ptr(out), int(nthreads), ctypes.byref(secs))
    if rc < 1:
        raise RuntimeError(f"oracle_jacobi2d_omp_timed failed rc={rc}")
    return out, rc, secs.value


def checksum(u: np.ndarray) -> float:
    nx, ny, nz = _dims(u)
    return lib().oracle_checksum(nx, ny, nz, _ptr(u))


def bithash(u: np.ndarray) -> int:
    nx, ny, nz = _dims(u)
    return int(lib().oracle_bithash(nx, ny, nz, _ptr(u)))
