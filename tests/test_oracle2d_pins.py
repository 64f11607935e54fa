"""Pins of the Jacobi2D oracle (NEXT-1) against things other than itself: constant
fixed point (fl(1/5) = (1/5)(1 + 2^-54) exactly, so 5c*K rounds back to c), harmonic
linear field on a non-square grid, the 3x3 hand case (golden/p3_square3_2d.txt),
separable eigenmode closed form, exact-rational bound, numpy second oracle, blockwise
partition invariance, OpenMP == serial."""
import os
from fractions import Fraction

import numpy as np
import pytest

import jac_inputs as J
import oracle
from oracle.oracle_np import jacobi2d_np, sweep2d_np

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
GAMMA5 = 5 * 2.0 ** -53 / (1 - 5 * 2.0 ** -53)


def test_k5_is_one_fifth_times_one_plus_2_pow_minus_54():
    k5 = Fraction(float.fromhex("0x1.999999999999ap-3"))
    assert k5 == Fraction(1, 5) * (1 + Fraction(1, 2 ** 54))


@pytest.mark.parametrize("c", [1.0, 3.25, 12345.0, -7.0, 2.0 ** -30, 99991.0])
def test_constant_fixed_point(c):
    u0 = np.full((7, 9), c)
    assert np.array_equal(oracle.jacobi2d(u0, 9), u0)


@pytest.mark.parametrize("dims", [(7, 5), (1, 1), (2, 9), (13, 3)])
def test_linear_field_preserved(dims):
    nx, ny = dims
    j, i = np.meshgrid(np.arange(ny + 2), np.arange(nx + 2), indexing="ij")
    u0 = (i + 3.0 * j).astype(np.float64)
    assert np.array_equal(oracle.jacobi2d(u0, 6), u0)


def test_hand_case_3x3():
    u0 = np.zeros((5, 5))
    u0[1:-1, 1:-1] = 1.0
    cls = lambda i, j: sum(1 for c in (i, j) if c in (0, 2))
    names = {0: "centre", 1: "edge", 2: "corner"}
    n = 0
    for line in open(os.path.join(GOLDEN, "p3_square3_2d.txt")):
        if line.startswith("#") or not line.strip():
            continue
        it, sel, val = line.split()
        inner = oracle.jacobi2d(u0, int(it))[1:-1, 1:-1]
        want = float(Fraction(val))
        if sel == "sum":
            assert abs(inner.sum() - want) <= 9 * int(it) * GAMMA5 * 9
        else:
            got = [inner[j, i] for j in range(3) for i in range(3) if names[cls(i, j)] == sel]
            assert got and all(abs(g - want) <= int(it) * GAMMA5 for g in got)
        n += 1
    assert n == 8


@pytest.mark.parametrize("dims,n", [((30, 30), 20), ((41, 17), 33)])
def test_eigenmode(dims, n):
    nx, ny = dims
    u0 = np.zeros((ny + 2, nx + 2))
    sx = np.sin(np.pi * np.arange(1, nx + 1) / (nx + 1))
    sy = np.sin(np.pi * np.arange(1, ny + 1) / (ny + 1))
    u0[1:-1, 1:-1] = sy[:, None] * sx[None, :]
    lam = (1 + 2 * np.cos(np.pi / (nx + 1)) + 2 * np.cos(np.pi / (ny + 1))) / 5
    u = oracle.jacobi2d(u0, n)
    assert np.abs(u - lam ** n * u0).max() / np.abs(u0).max() < 1e-12


def test_rounding_bound_vs_exact():
    nx, ny, n = 5, 4, 7
    u0 = J.hash_field2d(nx, ny, seed=3)
    A = [[Fraction(float(u0[j, i])) for i in range(nx + 2)] for j in range(ny + 2)]
    for _ in range(n):
        B = [row[:] for row in A]
        for j in range(1, ny + 1):
            for i in range(1, nx + 1):
                B[j][i] = (A[j][i] + A[j][i - 1] + A[j][i + 1] + A[j - 1][i] + A[j + 1][i]) * Fraction(1, 5)
        A = B
    got = oracle.jacobi2d(u0, n)
    worst = max(abs(Fraction(float(got[j, i])) - A[j][i]) for j in range(ny + 2) for i in range(nx + 2))
    assert 0 < float(worst) <= n * GAMMA5 * np.abs(u0).max()


@pytest.mark.parametrize("dims,n", [((12, 10), 3), ((1, 7), 4), ((33, 17), 6)])
def test_numpy_second_oracle(dims, n):
    u0 = J.hash_field2d(*dims, seed=2)
    assert np.array_equal(oracle.jacobi2d(u0, n), jacobi2d_np(u0, n))


def test_partition_invariance_and_openmp():
    u0 = J.hash_field2d(24, 18, seed=1)
    want = oracle.jacobi2d(u0, 5)
    glob = u0.copy()
    for _ in range(5):
        new = glob.copy()
        for by in range(3):
            for bx in range(4):
                y0, x0 = by * 6, bx * 6
                blk = sweep2d_np(glob[y0:y0 + 8, x0:x0 + 8].copy())
                new[y0 + 1:y0 + 7, x0 + 1:x0 + 7] = blk[1:-1, 1:-1]
        glob = new
    assert np.array_equal(glob, want)
    out, _ = oracle.jacobi2d_omp(u0, 5, nthreads=3)
    assert np.array_equal(out, want)


def test_hash_field2d_layout():
    u = J.hash_field2d(5, 3, seed=2)
    for (j, i) in [(0, 0), (2, 3), (4, 6)]:
        assert u[j, i] == J.hash_values(2, np.array([j * 7 + i]))[0]
