"""Host transfers through the device staging slabs (engine.cu staged_transfer):
jac_set_init_box scatters slabs of whole planes (3-D) or rows (2-D) into both buffers
and the x-ghost arrays; jac_get_field_box gathers the interiors back.  Forced tiny slabs
(JAC_STAGE_BYTES=1: one plane / row per slab, i.e. slabs that cut blocks and their ghost
layers) must give the oracle's bits in both row layouts, leave every cell outside the
local interiors untouched, and work from pinned memory."""
import numpy as np
import pytest

import jac_inputs as JI
import oracle
import paper_2605_12734_b200 as jb

pytestmark = pytest.mark.gpu


def _bits(a, b):
    bad = np.flatnonzero(a.view(np.uint64) != b.view(np.uint64))
    assert bad.size == 0, f"{bad.size} mismatches, first at {np.unravel_index(bad[0], a.shape)}"


@pytest.mark.parametrize("pitched", [False, True])
@pytest.mark.parametrize("slab", ["1", "20000", None])
@pytest.mark.parametrize("dense", [True, False])
@pytest.mark.parametrize("dims,blocks", [((64, 48, 40), (2, 3, 5)), ((32, 32, 32), (4, 4, 4)), ((40, 24, 9), (1, 1, 1))])
def test_staged_init_and_readback_3d(monkeypatch, pitched, slab, dense, dims, blocks):
    monkeypatch.setenv("JAC_EXPERIMENT", "1")
    if pitched:  # the sub-box path (multi-GPU partitions) on one GPU
        monkeypatch.setenv("JAC_STAGE_PITCHED", "1")
    if slab:
        monkeypatch.setenv("JAC_STAGE_BYTES", slab)
    if not dense:
        monkeypatch.setenv("JAC_NO_DENSE", "1")
    u0 = JI.hash_field(*dims, seed=7)
    with jb.Jacobi3D(dims, blocks) as s:
        s.set_init(u0)
        _bits(s.field(u0), u0)  # round trip before any sweep
        s.step(1)  # every ghost cell the scatter wrote is read once
        _bits(s.field(u0), oracle.jacobi3d(u0, 1))
        s.step(4)
        _bits(s.field(u0), oracle.jacobi3d(u0, 5))


def test_field_box_leaves_the_shell_untouched(monkeypatch):
    monkeypatch.setenv("JAC_EXPERIMENT", "1")
    monkeypatch.setenv("JAC_STAGE_BYTES", "1")
    dims = (48, 32, 16)
    u0 = JI.hash_field(*dims, seed=8)
    with jb.Jacobi3D(dims, (2, 2, 2)) as s:
        s.set_init(u0)
        s.step(3)
        box = np.full_like(u0, np.nan)
        s.field_box(box, (0, 0, 0))
    want = oracle.jacobi3d(u0, 3)
    _bits(box[1:-1, 1:-1, 1:-1], want[1:-1, 1:-1, 1:-1])
    shell = np.ones(box.shape, bool)
    shell[1:-1, 1:-1, 1:-1] = False
    assert np.isnan(box[shell]).all()


@pytest.mark.parametrize("pitched", [False, True])
@pytest.mark.parametrize("slab", ["1", None])
@pytest.mark.parametrize("dims,blocks", [((200, 90), (2, 3)), ((64, 64), (1, 1)), ((70, 33), (5, 3))])
def test_staged_init_and_readback_2d(monkeypatch, pitched, slab, dims, blocks):
    monkeypatch.setenv("JAC_EXPERIMENT", "1")
    if pitched:
        monkeypatch.setenv("JAC_STAGE_PITCHED", "1")
    if slab:
        monkeypatch.setenv("JAC_STAGE_BYTES", slab)
    u0 = JI.hash_field2d(*dims, seed=9)
    with jb.Jacobi2D(dims, blocks) as s:
        s.set_init(u0)
        _bits(s.field(u0), u0)
        s.step(6)
        _bits(s.field(u0), oracle.jacobi2d_omp(u0, 6)[0])


@pytest.mark.parametrize("mode", [None, "JAC_STAGE_PITCHED", "JAC_DIRECT"])
def test_pinned_host_buffers(monkeypatch, mode):
    """Pinned boxes: staged slabs (default), the kernel reading the host rows itself
    (partial rows, here forced by JAC_STAGE_PITCHED) and the zero-copy path both ways
    (JAC_DIRECT)."""
    if mode:
        monkeypatch.setenv("JAC_EXPERIMENT", "1")
        monkeypatch.setenv(mode, "1")
    torch = pytest.importorskip("torch")
    dims = (64, 64, 64)
    u0 = JI.hash_field(*dims, seed=10)
    hin = torch.empty(u0.shape, dtype=torch.float64, pin_memory=True).numpy()
    hin[...] = u0
    hout = torch.empty(u0.shape, dtype=torch.float64, pin_memory=True).numpy()
    hout[...] = 0.0
    with jb.Jacobi3D(dims, (2, 2, 2)) as s:
        s.set_init_box(hin, (0, 0, 0))
        s.step(2)
        s.field_box(hout, (0, 0, 0))
    _bits(hout[1:-1, 1:-1, 1:-1], oracle.jacobi3d(u0, 2)[1:-1, 1:-1, 1:-1])


@pytest.mark.parametrize("pitched", [False, True])
def test_interior_box_readback(monkeypatch, pitched):
    """jac_get_field_box into a box of exactly the interiors (the linear read-back) and
    into a box one cell short of them (JAC_EINVAL)."""
    monkeypatch.setenv("JAC_EXPERIMENT", "1")
    monkeypatch.setenv("JAC_STAGE_BYTES", "1")
    if pitched:
        monkeypatch.setenv("JAC_STAGE_PITCHED", "1")
    dims = (40, 24, 16)
    u0 = JI.hash_field(*dims, seed=11)
    with jb.Jacobi3D(dims, (2, 1, 2)) as s:
        s.set_init(u0)
        s.step(3)
        inner = np.full((dims[2], dims[1], dims[0]), np.nan)
        s.field_box(inner, (1, 1, 1))
        _bits(inner, oracle.jacobi3d(u0, 3)[1:-1, 1:-1, 1:-1])
        short = np.zeros((dims[2] - 1, dims[1], dims[0]))
        with pytest.raises(jb.jacobi3d.JacError):
            s.field_box(short, (1, 1, 1))


@pytest.mark.parametrize("seed", range(8))
def test_staged_transfer_fuzz(monkeypatch, seed):
    """Random shapes, block grids, slab sizes and copy paths (linear, pitched, zero-copy
    from pinned memory): init + read-back round trip and one sweep against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    monkeypatch.setenv("JAC_EXPERIMENT", "1")
    monkeypatch.setenv("JAC_STAGE_BYTES", str(int(rng.integers(1, 200000))))
    if rng.random() < 0.5:
        monkeypatch.setenv("JAC_STAGE_PITCHED", "1")
    blocks = tuple(int(b) for b in rng.integers(1, 4, size=3))
    dims = tuple(int(b * e) for b, e in zip(blocks, rng.integers(2, 12, size=3) * 2))
    u0 = JI.hash_field(*dims, seed=20 + seed)
    pinned = rng.random() < 0.5
    if pinned:
        torch = pytest.importorskip("torch")
        h = torch.empty(u0.shape, dtype=torch.float64, pin_memory=True).numpy()
        h[...] = u0
        u_in = h
    else:
        u_in = u0
    with jb.Jacobi3D(dims, blocks) as s:
        s.set_init_box(u_in, (0, 0, 0))
        _bits(s.field(u0), u0)
        s.step(1)
        _bits(s.field(u0), oracle.jacobi3d(u0, 1))


def test_pinned_x_split_group(monkeypatch):
    """One process, two GPUs split in x: each device's partial-row sub-box of one pinned
    host array takes the zero-copy init (the array was pinned by device 0's context)."""
    torch = pytest.importorskip("torch")
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    dims = (96, 40, 36)
    u0 = JI.hash_field(*dims, seed=31)
    h = torch.empty(u0.shape, dtype=torch.float64, pin_memory=True).numpy()
    h[...] = u0
    with jb.Jacobi3D(dims, (2, 1, 1), n_gpus=2, gpu_grid=(2, 1, 1)) as s:
        s.set_init_box(h, (0, 0, 0))
        _bits(s.field(u0), u0)
        s.step(3)
        _bits(s.field(u0), oracle.jacobi3d(u0, 3))
