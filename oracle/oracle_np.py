"""Second, independently written oracle in numpy -- TEST INFRASTRUCTURE ONLY (pin P6).

Whole-array slices instead of the C oracle's scalar loops; the per-point operation
order is the frozen reading of SURVEY.md §8(c) R2-R4:
``((((((c + x-) + x+) + y-) + y+) + z-) + z+) * fl(1/7)``, shell fixed (R6).
numpy float64 elementwise adds/multiplies are single IEEE operations, so this must
agree with the C oracle bit for bit.
"""
from __future__ import annotations

import numpy as np

K = float.fromhex("0x1.2492492492492p-3")  # fl(1/7), reading R3


def sweep_np(A: np.ndarray) -> np.ndarray:
    """One Jacobi sweep of the padded array A (shape [nz+2, ny+2, nx+2])."""
    B = A.copy()
    c = A[1:-1, 1:-1, 1:-1]
    s = c + A[1:-1, 1:-1, :-2]   # x-
    s = s + A[1:-1, 1:-1, 2:]    # x+
    s = s + A[1:-1, :-2, 1:-1]   # y-
    s = s + A[1:-1, 2:, 1:-1]    # y+
    s = s + A[:-2, 1:-1, 1:-1]   # z-
    s = s + A[2:, 1:-1, 1:-1]    # z+
    B[1:-1, 1:-1, 1:-1] = s * K
    return B


def jacobi3d_np(u0: np.ndarray, n: int) -> np.ndarray:
    A = np.array(u0, dtype=np.float64, copy=True)
    for _ in range(int(n)):
        A = sweep_np(A)
    return A


K5 = float.fromhex("0x1.999999999999ap-3")  # fl(1/5), 2-D reading


def sweep2d_np(A: np.ndarray) -> np.ndarray:
    """One 5-point sweep of the padded 2-D array A (shape [ny+2, nx+2])."""
    B = A.copy()
    s = A[1:-1, 1:-1] + A[1:-1, :-2]   # c + x-
    s = s + A[1:-1, 2:]                # x+
    s = s + A[:-2, 1:-1]               # y-
    s = s + A[2:, 1:-1]                # y+
    B[1:-1, 1:-1] = s * K5
    return B


def jacobi2d_np(u0: np.ndarray, n: int) -> np.ndarray:
    A = np.array(u0, dtype=np.float64, copy=True)
    for _ in range(int(n)):
        A = sweep2d_np(A)
    return A
