"""Row layouts: dense rows (3-D, ex % 8 == 0, the default) and the
padded rows (JAC_NO_DENSE=1, and every width that is not a multiple of 8) give the
oracle's bits; jac_get_block_padded returns the unstored x-edge ghost corners of the
dense layout as NaN and real values elsewhere."""
import numpy as np
import pytest

import jac_inputs as JI
import oracle
import paper_2605_12734_b200 as jb

pytestmark = pytest.mark.gpu


def _bits_equal(a, b):
    return np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("dense", [True, False])
@pytest.mark.parametrize("dims,blocks", [((64, 64, 64), (2, 2, 2)), ((128, 96, 80), (2, 2, 2)),
                                         ((512, 64, 48), (2, 2, 1)), ((48, 40, 24), (3, 1, 2))])
def test_both_layouts_bit_exact(monkeypatch, dense, dims, blocks):
    if not dense:
        monkeypatch.setenv("JAC_EXPERIMENT", "1")
        monkeypatch.setenv("JAC_NO_DENSE", "1")
    u0 = JI.hash_field(*dims, seed=2)
    with jb.Jacobi3D(dims, blocks) as s:
        s.set_init(u0)
        s.step(7)
        got = s.field(u0)
    assert _bits_equal(got, oracle.jacobi3d(u0, 7))


def test_hash_init_dense_matches_generator():
    """hash_init_kernel writes the x ghosts of dense rows straight into the x-ghost
    arrays: the first sweep must see the generator's values."""
    dims, blocks = (64, 48, 32), (2, 2, 2)
    u0 = JI.hash_field(*dims, seed=5)
    with jb.Jacobi3D(dims, blocks) as s:
        s.set_init_hash(5)
        s.step(3)
        got = s.field(u0)
    assert _bits_equal(got, oracle.jacobi3d(u0, 3))


def test_block_padded_corners():
    dims, blocks = (32, 24, 16), (2, 2, 2)  # ex = 16: dense rows
    u0 = JI.hash_field(*dims, seed=1)
    with jb.Jacobi3D(dims, blocks) as s:
        s.set_init(u0)
        ex, ey, ez = s.block_extent
        b = s.block_padded(1, 1, 1)
    want = u0[ez:2 * ez + 2, ey:2 * ey + 2, ex:2 * ex + 2]
    inner = b[:, :, 1:-1]  # every cell but the x ghost columns
    assert _bits_equal(inner, want[:, :, 1:-1])
    xcols = b[1:-1, 1:-1, [0, -1]]  # x ghosts of interior rows: from the x-ghost arrays
    assert _bits_equal(xcols, want[1:-1, 1:-1, [0, -1]])
    corners = np.concatenate([b[[0, -1], :, :][:, :, [0, -1]].ravel(), b[:, [0, -1], :][:, :, [0, -1]].ravel()])
    assert np.isnan(corners).all()


@pytest.mark.parametrize("pdl", ["0", "1"])
@pytest.mark.parametrize("dims,blocks,flags", [((64, 64, 64), (2, 2, 2), 0), ((128, 128, 128), (2, 2, 4), 0),
                                               ((256, 192, 1), (2, 2, 1), 1 << 9)])
def test_programmatic_dependent_launch_on_off(monkeypatch, pdl, dims, blocks, flags):
    """Sweeps with and without programmatic dependent launch (JAC_PDL) give the same
    bits: every CTA waits on griddepcontrol before touching a buffer."""
    monkeypatch.setenv("JAC_EXPERIMENT", "1")
    monkeypatch.setenv("JAC_PDL", pdl)
    if flags:
        u0 = JI.hash_field2d(dims[0], dims[1], seed=3)
        with jb.Jacobi2D(dims[:2], blocks[:2]) as s:
            s.set_init(u0)
            s.step(9)
            got = s.field(u0)
        assert _bits_equal(got, oracle.jacobi2d(u0, 9))
        return
    u0 = JI.hash_field(*dims, seed=3)
    with jb.Jacobi3D(dims, blocks) as s:
        s.set_init(u0)
        s.step(9)
        got = s.field(u0)
    assert _bits_equal(got, oracle.jacobi3d(u0, 9))
