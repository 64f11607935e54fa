"""Pins of the CPU oracle against things other than itself.

Every test here is -m "not gpu".  Each pin is chosen so that a plausible slip in
the oracle (a dropped term, a wrong sign or stride, a transposed axis, a different
summation order or a /7 instead of x fl(1/7)) fails at least one of them:

* dropped / duplicated term      -> P1 constant field, P3 hand cases
* wrong stride, sign or axis     -> P2 linear field on a non-cubic grid, P4 eigenmode
                                    on a non-cubic grid, P3-D (x-face only)
* wrong order / division by 7    -> C1 regression constants (independent survey code)
* shell handling                 -> P3 (zero shell), P2 (linear shell), P8 light cone
"""
from __future__ import annotations

import os
from fractions import Fraction

import numpy as np
import pytest

import jac_inputs as J
import oracle
from oracle.oracle_np import jacobi3d_np, sweep_np

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
U = 2.0 ** -53
GAMMA7 = 7 * U / (1 - 7 * U)


def _read_kv(name):
    out = {}
    for line in open(os.path.join(GOLDEN, name)):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        k, v = line.split(None, 1)
        out[k] = v
    return out


# ---------------------------------------------------------------- generator pins
def test_hash_init_pins():
    """R11 generator == SURVEY's independently computed values (golden/hash_init.txt)."""
    for line in open(os.path.join(GOLDEN, "hash_init.txt")):
        if line.startswith("#") or not line.strip():
            continue
        seed, p, val = line.split()
        got = float(J.hash_values(int(seed), np.array([int(p)]))[0])
        assert got == float.fromhex(val), (seed, p, got.hex(), val)


def test_hash_field_layout():
    """hash_field cell (k,j,i) uses padded index p=(k*(ny+2)+j)*(nx+2)+i (R11 key)."""
    nx, ny, nz = 5, 4, 3
    u = J.hash_field(nx, ny, nz, seed=2, chunk_planes=2)
    for (k, j, i) in [(0, 0, 0), (1, 2, 3), (4, 5, 6), (2, 0, 6)]:
        p = (k * (ny + 2) + j) * (nx + 2) + i
        assert u[k, j, i] == J.hash_values(2, np.array([p]))[0]
    assert u.min() >= 0.0 and u.max() < 1.0


# ---------------------------------------------------------------- P1 constant field
@pytest.mark.parametrize("c", [1.0, 3.25, 12345.0, 2.0 ** -30, -7.0, 99991.0])
def test_p1_constant_field_is_fixed_point(c):
    """7c is exact and K = (1/7)(1 - 2^-54) rounds 7c*K back to c."""
    u0 = J.constant_field(7, 5, 6, c)
    u = oracle.jacobi3d(u0, 9)
    assert np.array_equal(u, u0)


# ---------------------------------------------------------------- P2 linear field
@pytest.mark.parametrize("dims", [(6, 5, 7), (3, 9, 4), (1, 1, 1), (11, 2, 3)])
def test_p2_linear_field_preserved(dims):
    """u = i + 2j + 4k (distinct weights per axis) is harmonic for the 7-point mean
    and its integer sums are exact, so it stays bit-identical everywhere."""
    nx, ny, nz = dims
    u0 = J.linear_field(nx, ny, nz)
    assert np.array_equal(oracle.jacobi3d(u0, 5), u0)


def test_p2_linear_zero_shell_lightcone():
    """Zero-shell variant: points farther than n from the shell keep their value."""
    nx, ny, nz = 13, 11, 12
    n = 3
    u0 = J.linear_field(nx, ny, nz, zero_shell=True)
    u = oracle.jacobi3d(u0, n)
    lin = J.linear_field(nx, ny, nz)
    # interior index d (1-based padded) is at distance d from shell plane 0
    sl = (slice(n + 1, nz + 1 - n), slice(n + 1, ny + 1 - n), slice(n + 1, nx + 1 - n))
    assert np.array_equal(u[sl], lin[sl])
    assert not np.array_equal(u, lin)  # the shell itself is zero, so the rim changed


# ---------------------------------------------------------------- P3 4^3 hand cases
def _p3_expect():
    rows = []
    for line in open(os.path.join(GOLDEN, "p3_cube4.txt")):
        if line.startswith("#") or not line.strip():
            continue
        case, it, sel, val = line.split()
        rows.append((case, int(it), sel, Fraction(val)))
    return rows


def _cls(i, j, k):
    return sum(1 for c in (i, j, k) if c in (0, 3))


def test_p3_cube4_hand_cases():
    fields = {"A": J.ones_interior_field(4, 4, 4),
              "B": J.delta_field(4, 4, 4, (1, 1, 1)),
              "D": J.face_x_minus_field(4, 4, 4)}
    names = {0: "deep", 1: "face", 2: "edge", 3: "corner"}
    checked = 0
    for case, it, sel, val in _p3_expect():
        u = oracle.jacobi3d(fields[case], it)
        inner = u[1:-1, 1:-1, 1:-1]  # [k][j][i]
        tol = it * GAMMA7 * 1.0 * 64 + 1e-300  # P5 bound per point (||u0||=1), x64 for sums
        if sel in names.values():
            want = [float(val)]
            got = [inner[k, j, i] for k in range(4) for j in range(4) for i in range(4)
                   if names[_cls(i, j, k)] == sel]
            assert got and all(abs(g - want[0]) <= it * GAMMA7 for g in got), (case, it, sel)
        elif sel == "sum":
            assert abs(inner.sum() - float(val)) <= tol, (case, it, sel)
        elif sel == "nnz":
            assert int(np.count_nonzero(inner)) == int(val), (case, it)
        elif sel == "nonzero":
            nz = inner[inner != 0]
            assert np.all(np.abs(nz - float(val)) <= it * GAMMA7)
        elif sel.startswith("plane_x"):
            x = int(sel[-1])
            assert np.all(np.abs(inner[:, :, x] - float(val)) <= it * GAMMA7), (case, it, sel)
        elif sel.startswith("at_"):
            i, j, k = map(int, sel[3:].split("_"))
            assert abs(inner[k, j, i] - float(val)) <= it * GAMMA7, (case, it, sel)
        else:
            raise AssertionError(sel)
        checked += 1
    assert checked == 26


# ---------------------------------------------------------------- P4 eigenmode
@pytest.mark.parametrize("dims,n", [((24, 24, 24), 10), ((20, 13, 9), 25), ((64, 64, 64), 100)])
def test_p4_eigenmode_closed_form(dims, n):
    """u0 = prod sin(pi (i+1)/(N+1)), zero shell => u_n = lambda^n u0 with
    lambda = (1 + 2 cos(pi/(Nx+1)) + 2 cos(pi/(Ny+1)) + 2 cos(pi/(Nz+1))) / 7."""
    nx, ny, nz = dims
    u0 = J.eigenmode_field(nx, ny, nz)
    lam = (1 + 2 * np.cos(np.pi / (nx + 1)) + 2 * np.cos(np.pi / (ny + 1))
           + 2 * np.cos(np.pi / (nz + 1))) / 7
    u = oracle.jacobi3d(u0, n)
    want = lam ** n * u0
    err = np.abs(u - want).max() / np.abs(want).max()
    assert err < 1e-12, err


# ---------------------------------------------------------------- P5 rounding bound
def test_p5_rounding_bound_vs_exact_rationals():
    """Brute force in exact rationals (1/7 exact) on a random 4x5x3 grid:
    |oracle - exact|_inf <= n * gamma_7 * ||u0||_inf for non-negative data."""
    nx, ny, nz, n = 4, 5, 3, 6
    u0 = J.hash_field(nx, ny, nz, seed=3)
    A = [[[Fraction(float(u0[k, j, i])) for i in range(nx + 2)] for j in range(ny + 2)]
         for k in range(nz + 2)]
    seven = Fraction(1, 7)
    for _ in range(n):
        B = [[row[:] for row in plane] for plane in A]
        for k in range(1, nz + 1):
            for j in range(1, ny + 1):
                for i in range(1, nx + 1):
                    B[k][j][i] = (A[k][j][i] + A[k][j][i - 1] + A[k][j][i + 1] + A[k][j - 1][i]
                                  + A[k][j + 1][i] + A[k - 1][j][i] + A[k + 1][j][i]) * seven
        A = B
    got = oracle.jacobi3d(u0, n)
    bound = n * GAMMA7 * float(np.abs(u0).max())
    worst = max(abs(Fraction(float(got[k, j, i])) - A[k][j][i])
                for k in range(nz + 2) for j in range(ny + 2) for i in range(nx + 2))
    assert float(worst) <= bound, (float(worst), bound)
    assert float(worst) > 0  # the oracle does round (it is not secretly exact)


# ---------------------------------------------------------------- P6 numpy second oracle
@pytest.mark.parametrize("dims,n", [((12, 10, 8), 3), ((1, 7, 2), 4), ((33, 5, 17), 6)])
def test_p6_numpy_oracle_bit_identical(dims, n):
    u0 = J.hash_field(*dims, seed=2)
    assert np.array_equal(oracle.jacobi3d(u0, n), jacobi3d_np(u0, n))


# ---------------------------------------------------------------- P7 partition invariance
def _blockwise(u0, blocks, n):
    """CPU blockwise Jacobi: each block is a ghosted copy updated on its own and
    refreshed from its neighbours' interiors after every sweep."""
    nz2, ny2, nx2 = u0.shape
    nx, ny, nz = nx2 - 2, ny2 - 2, nz2 - 2
    bx, by, bz = blocks
    ex, ey, ez = nx // bx, ny // by, nz // bz
    glob = u0.copy()
    for _ in range(n):
        new = glob.copy()
        for kz in range(bz):
            for ky in range(by):
                for kx in range(bx):
                    z0, y0, x0 = kz * ez, ky * ey, kx * ex
                    blk = glob[z0:z0 + ez + 2, y0:y0 + ey + 2, x0:x0 + ex + 2].copy()
                    out = sweep_np(blk)
                    new[z0 + 1:z0 + ez + 1, y0 + 1:y0 + ey + 1, x0 + 1:x0 + ex + 1] = \
                        out[1:-1, 1:-1, 1:-1]
        glob = new
    return glob


@pytest.mark.parametrize("blocks", [(2, 2, 2), (3, 1, 2), (1, 4, 1)])
def test_p7_partition_invariance_cpu(blocks):
    u0 = J.hash_field(12, 8, 10, seed=1)
    assert np.array_equal(_blockwise(u0, blocks, 3), oracle.jacobi3d(u0, 3))


# ---------------------------------------------------------------- P8 light cone
def test_p8_light_cone_subcube():
    """A sub-cube after n sweeps depends only on the cube grown by n cells (clipped
    at the global shell); the oracle run on that region with its ring frozen
    reproduces the global result bit for bit."""
    nx = ny = nz = 40
    n = 6
    u0 = J.hash_field(nx, ny, nz, seed=1)
    full = oracle.jacobi3d(u0, n)
    for (x0, y0, z0, s) in [(0, 0, 0, 8), (17, 9, 22, 10), (32, 30, 31, 8)]:
        lo = [max(0, c - n) for c in (z0, y0, x0)]           # interior 0-based
        hi = [min(N, c + s + n) for c, N in ((z0, nz), (y0, ny), (x0, nx))]
        sub = u0[lo[0]:hi[0] + 2, lo[1]:hi[1] + 2, lo[2]:hi[2] + 2].copy()
        res = oracle.jacobi3d(sub, n)
        a = res[z0 - lo[0] + 1:z0 - lo[0] + 1 + s, y0 - lo[1] + 1:y0 - lo[1] + 1 + s,
                x0 - lo[2] + 1:x0 - lo[2] + 1 + s]
        b = full[z0 + 1:z0 + 1 + s, y0 + 1:y0 + 1 + s, x0 + 1:x0 + 1 + s]
        assert np.array_equal(a, b)


# ---------------------------------------------------------------- P9 identity / restart
def test_p9_identity_determinism_restart():
    u0 = J.hash_field(9, 7, 8, seed=3)
    assert np.array_equal(oracle.jacobi3d(u0, 0), u0)
    a = oracle.jacobi3d(u0, 7)
    assert np.array_equal(a, oracle.jacobi3d(u0, 7))
    assert np.array_equal(oracle.jacobi3d(oracle.jacobi3d(u0, 3), 4), a)
    assert oracle.bithash(a) == oracle.bithash(a.copy())


# ---------------------------------------------------------------- P10 threaded == serial
def test_p10_openmp_equals_serial():
    u0 = J.hash_field(80, 40, 64, seed=2)
    out, threads = oracle.jacobi3d_omp(u0, 4, nthreads=4)
    assert np.array_equal(out, oracle.jacobi3d(u0, 4))
    assert oracle.lib().oracle_has_openmp() == 1


# ---------------------------------------------------------------- P12 max principle
def test_p12_max_principle():
    u0 = J.hash_field(20, 18, 16, seed=1)
    n = 12
    u = oracle.jacobi3d(u0, n)
    M = np.abs(u0).max()
    assert u.min() >= u0.min() - n * GAMMA7 * M
    assert u.max() <= u0.max() + n * GAMMA7 * M


# ---------------------------------------------------------------- C1 regression
def test_c1_regression_constants():
    """BASELINE.json configs[0]: 64^3, seed-1 hash, 10 iterations.  Constants from the
    survey's independent numpy and scalar C++ codes (golden/c1_regression.txt)."""
    g = _read_kv("c1_regression.txt")
    nx, ny, nz = int(g["nx"]), int(g["ny"]), int(g["nz"])
    u0 = J.hash_field(nx, ny, nz, seed=int(g["seed"]))
    assert oracle.checksum(u0) == float.fromhex(g["checksum_iter0"])
    assert oracle.bithash(u0) == int(g["bithash_iter0"], 16)
    u = oracle.jacobi3d(u0, int(g["iters"]))
    assert oracle.checksum(u) == float.fromhex(g["checksum"])
    assert oracle.bithash(u) == int(g["bithash"], 16)
    assert u[1, 1, 1] == float.fromhex(g["u_interior_0_0_0"])


def test_oracle_rejects_bad_args():
    L = oracle.lib()
    assert L.oracle_jacobi3d(0, 1, 1, None, 1, None) == -1
    with pytest.raises(ValueError):
        oracle.jacobi3d(np.zeros((3, 3, 3), dtype=np.float32), 1)
