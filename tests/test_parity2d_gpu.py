"""Jacobi2D (NEXT-1) GPU parity: the 2-D TMA sweep through the C ABI (JAC_F_2D) vs
the 2-D CPU oracle, bit for bit, for every block decomposition ("bit-exact
... serial reference Jacobi on the full grid", SPEC.md:482 partition invariance)."""
import numpy as np
import pytest

import jac_inputs as JI
import oracle
import paper_2605_12734_b200 as jb
from paper_2605_12734_b200 import jacobi3d as J

pytestmark = pytest.mark.gpu


def ref(u0, n):
    return oracle.jacobi2d_omp(u0, n)[0]


def run(u0, blocks, n, n_gpus=1, flags=0, steps=None):
    ny2, nx2 = u0.shape
    with jb.Jacobi2D((nx2 - 2, ny2 - 2), blocks, n_gpus=n_gpus, flags=flags) as s:
        s.set_init(u0)
        for k in (steps or [n]):
            s.step(k)
        return s.field(u0)


def bits(a, b):
    bad = np.flatnonzero(a.view(np.uint64) != b.view(np.uint64))
    assert bad.size == 0, f"{bad.size} mismatches, first {np.unravel_index(bad[0], a.shape)}"


@pytest.mark.parametrize("dims,blocks", [((256, 192), (1, 1)), ((256, 192), (2, 3)), ((256, 192), (4, 4)),
                                         ((100, 37), (2, 1)), ((70, 33), (5, 3)), ((1, 1), (1, 1)),
                                         ((64, 64), (2, 2)), ((512, 96), (8, 2)), ((130, 2), (2, 2))])
def test_2d_decompositions(dims, blocks):
    u0 = JI.hash_field2d(*dims, seed=1)
    bits(run(u0, blocks, 9), ref(u0, 9))


def test_2d_step_chunks_and_virtual_partitions():
    u0 = JI.hash_field2d(192, 128, seed=2)
    want = ref(u0, 23)
    bits(run(u0, (4, 2), 23, steps=[1, 10, 12]), want)
    bits(run(u0, (4, 4), 23, n_gpus=4, flags=J.JAC_F_VIRTUAL_GPUS), want)


def test_2d_device_hash_init_and_structured_fields():
    nx, ny = 96, 40
    u0 = JI.hash_field2d(nx, ny, seed=3)
    with jb.Jacobi2D((nx, ny), (2, 2)) as s:
        s.set_init_hash(3)
        bits(s.block_padded(1, 1), u0[20:42, 48:98])
        s.step(5)
        bits(s.field(u0), ref(u0, 5))
    c = np.full((12, 20), 3.25)
    bits(run(c, (2, 2), 7), c)


def test_2d_rejects_3d_shapes_and_flags():
    with pytest.raises(J.JacError):
        jb.Jacobi3D((8, 8, 2), (1, 1, 1), flags=J.JAC_F_2D)
    with pytest.raises(J.JacError):
        jb.Jacobi2D((8, 8), (1, 1), flags=J.JAC_F_NO_TMA)


@pytest.mark.parametrize("threads", [1, 4])
@pytest.mark.parametrize("dims,blocks", [((256, 192), (4, 3)), ((130, 66), (2, 2)), ((64, 64), (1, 1))])
def test_2d_paper_style_per_block_mode(threads, dims, blocks):
    """NEXT-2 on the paper's own app: per-block streams, per-face pack / unpack
    launches, several launching threads -- bit-identical to the 2-D oracle."""
    u0 = JI.hash_field2d(*dims, seed=1)
    with jb.Jacobi2D(dims, blocks, flags=J.JAC_F_PER_BLOCK) as s:
        s.set_option(J.JAC_OPT_LAUNCH_THREADS, threads)
        s.set_init(u0)
        s.step(4)
        s.step(5)
        bits(s.field(u0), ref(u0, 9))


@pytest.mark.parametrize("band", ["1", "3", "5"])
def test_2d_x_bands(monkeypatch, band):
    """The 2-D work list in x bands (decode_item2d; default 512 tiles, so only blocks
    wider than 32768 points use more than one): forced narrow bands, including a ragged
    last band, keep every item exactly once -- plain, in blocks, and with virtual
    partitions (remote items spread by the item map)."""
    monkeypatch.setenv("JAC_EXPERIMENT", "1")
    monkeypatch.setenv("JAC_XBAND", band)
    u0 = JI.hash_field2d(1000, 300, seed=4)  # 16 x tiles of 64 (ragged last tile)
    want = ref(u0, 7)
    bits(run(u0, (1, 1), 7), want)
    bits(run(u0, (2, 3), 7), want)
    bits(run(u0, (2, 2), 7, n_gpus=4, flags=J.JAC_F_VIRTUAL_GPUS), want)
