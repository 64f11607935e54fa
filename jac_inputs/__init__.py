"""Seeded synthetic input fields for the Jacobi3D hot path.

This module is the ONLY code shared by the oracle side (tests/, oracle/) and the
CUDA side (tests feeding ``jac_set_init``; bench.py).  It holds no arithmetic of the
method -- only initial fields on the padded grid ``[nz+2, ny+2, nx+2]`` (x fastest,
reading R7: nx, ny, nz count updated points, the Dirichlet shell is extra).

* ``hash_field`` -- SURVEY.md §8(c.2) R11: counter-based splitmix64 of
  ``key = (seed << 40) + p`` (p = padded linear index), ``u = (h >> 11) * 2^-53``.
  The CUDA library implements the same generator on the device
  (``jac_set_init_hash``); both are pinned to the values in
  tests/golden/hash_init.txt.
* structured correctness fields (constant, linear, eigenmode, delta, face) --
  SURVEY.md §8(c.3) pins P1-P4.

Workload recipe: the paper's Jacobi runs use a uniform dense grid,
a fixed iteration count and no convergence check; values do not
affect the branch-free kernel, so benches use ``hash_field(seed=1)``.
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (mod 2^64)."""
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z += np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def hash_values(seed: int, p: np.ndarray) -> np.ndarray:
    """R11 value of padded cell(s) p for ``seed``: uniform in [0, 1)."""
    key = (np.uint64(seed) << np.uint64(40)) + np.asarray(p, dtype=np.uint64)
    h = splitmix64(key)
    return (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def hash_field(nx: int, ny: int, nz: int, seed: int = 1, chunk_planes: int = 64) -> np.ndarray:
    """Padded R11 hash field, shell included."""
    u = np.empty((nz + 2, ny + 2, nx + 2), dtype=np.float64)
    plane = (ny + 2) * (nx + 2)
    for k0 in range(0, nz + 2, chunk_planes):
        k1 = min(nz + 2, k0 + chunk_planes)
        p = np.arange(k0 * plane, k1 * plane, dtype=np.uint64)
        u[k0:k1] = hash_values(seed, p).reshape(k1 - k0, ny + 2, nx + 2)
    return u


def hash_box(nx: int, ny: int, nz: int, origin, extent, seed: int = 1) -> np.ndarray:
    """Sub-box [extent z, y, x] of the padded R11 hash field starting at padded cell
    origin = (ox, oy, oz) -- what one rank of a multi-GPU run holds."""
    ox, oy, oz = (int(v) for v in origin)
    sx, sy, sz = (int(v) for v in extent)
    u = np.empty((sz, sy, sx), dtype=np.float64)
    xs = np.arange(ox, ox + sx, dtype=np.uint64)
    for k in range(sz):
        rows = (np.uint64(oz + k) * np.uint64(ny + 2) + np.arange(oy, oy + sy, dtype=np.uint64))
        p = rows[:, None] * np.uint64(nx + 2) + xs[None, :]
        u[k] = hash_values(seed, p)
    return u


def hash_field2d(nx: int, ny: int, seed: int = 1) -> np.ndarray:
    """Padded 2-D R11 hash field [ny+2, nx+2]: key (seed << 40) + p, p = j*(nx+2) + i."""
    p = np.arange((ny + 2) * (nx + 2), dtype=np.uint64)
    return hash_values(seed, p).reshape(ny + 2, nx + 2)


def constant_field(nx: int, ny: int, nz: int, c: float) -> np.ndarray:
    """P1: every padded cell = c."""
    return np.full((nz + 2, ny + 2, nx + 2), c, dtype=np.float64)


def linear_field(nx: int, ny: int, nz: int, a=(1.0, 2.0, 4.0), zero_shell: bool = False) -> np.ndarray:
    """P2: u = a0*i + a1*j + a2*k on padded coordinates (shell included)."""
    k, j, i = np.meshgrid(np.arange(nz + 2), np.arange(ny + 2), np.arange(nx + 2), indexing="ij")
    u = (a[0] * i + a[1] * j + a[2] * k).astype(np.float64)
    if zero_shell:
        u[0, :, :] = u[-1, :, :] = 0.0
        u[:, 0, :] = u[:, -1, :] = 0.0
        u[:, :, 0] = u[:, :, -1] = 0.0
    return u


def eigenmode_field(nx: int, ny: int, nz: int) -> np.ndarray:
    """P4: prod_d sin(pi (i_d+1) / (N_d+1)) on the interior (0-based i_d), zero shell."""
    u = np.zeros((nz + 2, ny + 2, nx + 2), dtype=np.float64)
    sx = np.sin(np.pi * np.arange(1, nx + 1) / (nx + 1))
    sy = np.sin(np.pi * np.arange(1, ny + 1) / (ny + 1))
    sz = np.sin(np.pi * np.arange(1, nz + 1) / (nz + 1))
    u[1:-1, 1:-1, 1:-1] = sz[:, None, None] * sy[None, :, None] * sx[None, None, :]
    return u


def delta_field(nx: int, ny: int, nz: int, at=(1, 1, 1)) -> np.ndarray:
    """P3-B: 1 at interior point ``at`` = (i, j, k) 0-based, zero elsewhere."""
    u = np.zeros((nz + 2, ny + 2, nx + 2), dtype=np.float64)
    i, j, k = at
    u[k + 1, j + 1, i + 1] = 1.0
    return u


def ones_interior_field(nx: int, ny: int, nz: int) -> np.ndarray:
    """P3-A: interior ones, shell zero."""
    u = np.zeros((nz + 2, ny + 2, nx + 2), dtype=np.float64)
    u[1:-1, 1:-1, 1:-1] = 1.0
    return u


def face_x_minus_field(nx: int, ny: int, nz: int) -> np.ndarray:
    """P3-D: shell face x = -1 set to 1 (its edges/corners 0), everything else 0."""
    u = np.zeros((nz + 2, ny + 2, nx + 2), dtype=np.float64)
    u[1:-1, 1:-1, 0] = 1.0
    return u
