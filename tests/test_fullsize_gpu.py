"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(device hash init, the bench's block shapes, 100 iterations): sampled outputs the
oracle computes one by one through the light cone (SURVEY.md §8(c.3) P8 -- a sub-cube
after n sweeps depends only on the cube grown by n cells, clipped at the shell), plus
bit-identity of sampled regions across ODFs.  Regions are read with jac_get_region."""
import numpy as np
import pytest

import jac_inputs as JI
import oracle
import paper_2605_12734_b200 as jb
from paper_2605_12734_b200 import jacobi3d as J

pytestmark = pytest.mark.gpu
N_IT = 100


def lightcone3d(dims, n, lo, s, seed=1):
    nx, ny, nz = dims
    a = [max(0, lo[d] - n) for d in range(3)]
    b = [min(dims[d], lo[d] + s + n) for d in range(3)]
    sub = JI.hash_box(nx, ny, nz, origin=a, extent=[b[d] - a[d] + 2 for d in range(3)], seed=seed)
    res, _ = oracle.jacobi3d_omp(sub, n)
    return res[lo[2] - a[2] + 1:lo[2] - a[2] + 1 + s, lo[1] - a[1] + 1:lo[1] - a[1] + 1 + s,
               lo[0] - a[0] + 1:lo[0] - a[0] + 1 + s]


def bits(a, b):
    assert a.shape == b.shape
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def run_probes(dims, blocks, probes, s=8, compare=None):
    """Runs the bench configuration, checks light-cone probes; returns big-region values."""
    out = {}
    with jb.Jacobi3D(dims, blocks) as J3:
        J3.set_init_hash(1)
        J3.step(N_IT)
        for lo in probes:
            bits(J3.region(lo, (s, s, s)), lightcone3d(dims, N_IT, lo, s))
        if compare:
            out = {k: J3.region(*v) for k, v in compare.items()}
    return out


def test_c3_768_odf8_full_size():
    """BASELINE configs[2] per-GPU box: 768^3, ODF 8 (384^3 blocks), bench shapes."""
    dims = (768, 768, 768)
    probes = [(0, 0, 0), (380, 380, 380), (760, 760, 760), (383, 100, 700), (500, 383, 383)]
    cmp = {"seam": ((352, 352, 352), (64, 64, 64))}
    a = run_probes(dims, (2, 2, 2), probes, compare=cmp)
    b = run_probes(dims, (1, 1, 1), [], compare=cmp)
    bits(a["seam"], b["seam"])


def test_c4_1536_odf16_full_size():
    """BASELINE configs[3] at 1 GPU: 1536^3 (55 GB of HBM), ODF 16 (768x768x384 blocks)."""
    dims = (1536, 1536, 1536)
    probes = [(0, 0, 0), (764, 764, 380), (1528, 1528, 1528), (767, 1000, 383), (300, 767, 1151)]
    run_probes(dims, (2, 2, 4), probes)


def test_c5_shape_32cubed_blocks_full_size():
    """BASELINE configs[4]'s grid and block shape on one GPU: 1024^3 in 32^3 blocks
    (32768 blocks = 4096 per GPU at 8 GPUs), the fine-grain stress decomposition."""
    dims = (1024, 1024, 1024)
    probes = [(28, 28, 28), (508, 508, 508), (1016, 1016, 1016), (31, 511, 992)]
    cmp = {"blocks": ((60, 60, 60), (72, 72, 72))}
    a = run_probes(dims, (32, 32, 32), probes, compare=cmp)
    b = run_probes(dims, (2, 2, 2), [], compare=cmp)
    bits(a["blocks"], b["blocks"])


def test_j2d_32768_full_size():
    """NEXT-1 at the paper's Jacobi2D per-GPU size: 32768^2, ODF 8."""
    nx = ny = 32768
    n, s = N_IT, 16
    with jb.Jacobi2D((nx, ny), (2, 4)) as J2:
        J2.set_init_hash(1)
        J2.step(n)
        for (x0, y0) in [(0, 0), (16376, 8184), (32752, 32752), (16383, 24570)]:
            got = J2.region((x0, y0, 0), (s, s, 1))[0]
            a = [max(0, x0 - n), max(0, y0 - n)]
            b = [min(nx, x0 + s + n), min(ny, y0 + s + n)]
            ys = np.arange(a[1], b[1] + 2, dtype=np.uint64)[:, None]
            xs = np.arange(a[0], b[0] + 2, dtype=np.uint64)[None, :]
            sub = JI.hash_values(1, ys * np.uint64(nx + 2) + xs)
            res, _ = oracle.jacobi2d_omp(np.ascontiguousarray(sub), n)
            bits(got, res[y0 - a[1] + 1:y0 - a[1] + 1 + s, x0 - a[0] + 1:x0 - a[0] + 1 + s])


# ---------------------------------------------------------------- full memcmp
C2_ODF_BLOCKS = {1: (1, 1, 1), 2: (1, 1, 2), 4: (1, 2, 2), 8: (2, 2, 2), 16: (2, 2, 4), 32: (2, 4, 4),
                 64: (4, 4, 4), 512: (8, 8, 8), 4096: (16, 16, 16)}


def _full_run(dims, blocks, n, like):
    with jb.Jacobi3D(dims, blocks) as s:
        s.set_init_hash(1)
        s.step(n)
        return s.field(like)


def test_c2_full_memcmp_every_odf():
    """BASELINE configs[1] in full: 512^3, device hash init, 100 iterations, every ODF of
    the bench sweep (R9 block shapes) plus 64^3 and 32^3 blocks (C5's block shape) --
    the whole padded array equals the OpenMP oracle's bit for bit."""
    dims = (512, 512, 512)
    u0 = JI.hash_field(*dims, seed=1)
    want, _ = oracle.jacobi3d_omp(u0, N_IT)
    wv = want.view(np.uint64)
    for odf, blocks in C2_ODF_BLOCKS.items():
        got = _full_run(dims, blocks, N_IT, u0)
        bad = np.argwhere(got.view(np.uint64) != wv)
        assert len(bad) == 0, (f"ODF {odf} blocks {blocks}: {len(bad)} mismatches; bounding box (z, y, x) "
                               f"{bad.min(axis=0).tolist()} .. {bad.max(axis=0).tolist()}")
        del got


def test_c3x1_full_memcmp():
    """BASELINE configs[2] at one GPU in full: 768^3, ODF 8 (384^3 blocks), 100 iterations."""
    dims = (768, 768, 768)
    u0 = JI.hash_field(*dims, seed=1)
    want, _ = oracle.jacobi3d_omp(u0, N_IT)
    got = _full_run(dims, (2, 2, 2), N_IT, u0)
    bad = np.argwhere(got.view(np.uint64) != want.view(np.uint64))
    assert len(bad) == 0, (f"{len(bad)} mismatches; bounding box (z, y, x) {bad.min(axis=0).tolist()} .. "
                           f"{bad.max(axis=0).tolist()}; first {bad[:3].tolist()}")


def test_j2d_strong_paper_grid_multi_gpu():
    """NEXT-1 strong scaling at the paper's fixed grid, 131072 x 98304:
    two 103 GB fp64 arrays, so >= 2 B200 through jac_create(n_gpus=2) (one process);
    light-cone probes at the GPU seam, block seams and the corners after 100 iterations."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (206 GB of state)")
    nx, ny = 131072, 98304
    n, s = N_IT, 16
    with jb.Jacobi2D((nx, ny), (4, 4), n_gpus=2) as J2:
        assert J2.gpu_grid[:2] == (2, 1)
        J2.set_init_hash(1)
        J2.step(n)
        for (x0, y0) in [(0, 0), (65528, 49144), (65536, 0), (32760, 24568), (131056, 98288), (98300, 73720)]:
            got = J2.region((x0, y0, 0), (s, s, 1))[0]
            a = [max(0, x0 - n), max(0, y0 - n)]
            b = [min(nx, x0 + s + n), min(ny, y0 + s + n)]
            ys = np.arange(a[1], b[1] + 2, dtype=np.uint64)[:, None]
            xs = np.arange(a[0], b[0] + 2, dtype=np.uint64)[None, :]
            sub = JI.hash_values(1, ys * np.uint64(nx + 2) + xs)
            res, _ = oracle.jacobi2d_omp(np.ascontiguousarray(sub), n)
            bits(got, res[y0 - a[1] + 1:y0 - a[1] + 1 + s, x0 - a[0] + 1:x0 - a[0] + 1 + s])
