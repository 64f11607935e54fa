"""GPU parity: the CUDA path through the C ABI against the CPU oracle, element by
element, bit-exact (north star: "GPU results must be bit-exact to the oracle ...
the same across all ODFs"; the result is unique to the bit).

All inputs come from jac_inputs (seeded, synthetic, shaped like the paper's
Jacobi runs: uniform dense grid, fixed iteration count).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import jac_inputs as JI
import oracle
import paper_2605_12734_b200 as jb
from paper_2605_12734_b200 import jacobi3d as J

pytestmark = pytest.mark.gpu

F = J


def ref(u0, n):
    out, _ = oracle.jacobi3d_omp(u0, n)
    return out


def run(u0, blocks, n, flags=0, n_gpus=1, steps=None):
    nz2, ny2, nx2 = u0.shape
    with jb.Jacobi3D((nx2 - 2, ny2 - 2, nz2 - 2), blocks, n_gpus=n_gpus, flags=flags) as s:
        s.set_init(u0)
        for k in (steps or [n]):
            s.step(k)
        assert s.iterations == n
        return s.field(u0)


def assert_bits(a, b):
    assert a.shape == b.shape
    bad = np.flatnonzero(a.view(np.uint64) != b.view(np.uint64))
    assert bad.size == 0, f"{bad.size} mismatches, first at {np.unravel_index(bad[0], a.shape)}: {a.flat[bad[0]]!r} vs {b.flat[bad[0]]!r}"


def test_native_library_loaded():
    jb.load()
    maps = open("/proc/self/maps").read()
    assert J.lib_path() in maps


def test_c1_config_bit_exact_and_regression_constants():
    """BASELINE.json configs[0]: 64^3, 2x2x2 blocks (ODF 8), 1 GPU, 10 iterations."""
    u0 = JI.hash_field(64, 64, 64, seed=1)
    got = run(u0, (2, 2, 2), 10)
    assert_bits(got, ref(u0, 10))
    assert oracle.bithash(got) == 0x77818AA80EA02999  # tests/golden/c1_regression.txt


def test_device_hash_init_matches_generator():
    nx, ny, nz = 40, 24, 16
    u0 = JI.hash_field(nx, ny, nz, seed=3)
    with jb.Jacobi3D((nx, ny, nz), (2, 1, 2)) as s:
        s.set_init_hash(3)
        for iz in range(2):
            for ix in range(2):
                ex, ey, ez = s.block_extent
                blk = s.block_padded(ix, 0, iz)
                want = u0[iz * ez:iz * ez + ez + 2, 0:ey + 2, ix * ex:ix * ex + ex + 2]
                assert_bits(blk, want)
        s.step(4)
        assert_bits(s.field(u0), ref(u0, 4))


@pytest.mark.parametrize("blocks", [(1, 1, 1), (1, 1, 2), (1, 2, 2), (2, 2, 2), (2, 2, 4),
                                    (2, 4, 4), (4, 4, 4), (4, 8, 8)])
def test_odf_sweep_128(blocks):
    """ODF 1..256 at 128^3 (the C2 sweep's shapes, scaled down) all equal the oracle."""
    u0 = JI.hash_field(128, 128, 128, seed=2)
    want = ref(u0, 7)
    assert_bits(run(u0, blocks, 7), want)


@pytest.mark.parametrize("dims,blocks", [
    ((70, 37, 23), (2, 1, 1)),    # odd x extent 35, ragged tiles in x and y
    ((70, 37, 23), (5, 1, 1)),    # ex = 14: narrow tile variant
    ((33, 5, 9), (1, 1, 3)),      # odd everything, ez = 3
    ((130, 18, 6), (2, 2, 6)),    # ez = 1: every plane is a z-face
    ((1, 1, 1), (1, 1, 1)),
    ((2, 3, 4), (2, 3, 4)),       # 1^3 blocks: every point is a face point of 6 faces
    ((96, 66, 40), (3, 3, 5)),    # ex = 32 boundary of the narrow variant
])
def test_ragged_and_degenerate(dims, blocks):
    u0 = JI.hash_field(*dims, seed=1)
    assert_bits(run(u0, blocks, 5), ref(u0, 5))


@pytest.mark.parametrize("flags", [J.JAC_F_NO_TMA, J.JAC_F_UNFUSED_PACK, J.JAC_F_NO_GRAPH,
                                   J.JAC_F_UNFUSED_PACK | J.JAC_F_NO_TMA, J.JAC_F_FMA])
@pytest.mark.parametrize("dims,blocks", [((64, 48, 40), (2, 3, 2)), ((37, 21, 19), (1, 1, 1))])
def test_variants_bit_exact(flags, dims, blocks):
    u0 = JI.hash_field(*dims, seed=2)
    assert_bits(run(u0, blocks, 6, flags=flags), ref(u0, 6))


@pytest.mark.parametrize("n_gpus,blocks", [(2, (2, 2, 2)), (4, (2, 2, 4)), (8, (4, 4, 4)), (8, (2, 2, 2))])
def test_virtual_partitions(n_gpus, blocks):
    """Partition/REMOTE-face logic with all partitions on one device, one kernel."""
    u0 = JI.hash_field(64, 64, 64, seed=1)
    assert_bits(run(u0, blocks, 9, n_gpus=n_gpus, flags=J.JAC_F_VIRTUAL_GPUS), ref(u0, 9))


def test_step_accumulation_and_graph_unroll_boundaries():
    u0 = JI.hash_field(48, 40, 36, seed=3)
    want = ref(u0, 23)
    assert_bits(run(u0, (2, 2, 2), 23, steps=[0, 3, 10, 1, 9]), want)
    assert_bits(run(u0, (2, 2, 2), 23, steps=[23]), want)
    assert_bits(run(u0, (1, 1, 1), 0, steps=[0]), u0)


def test_restart_from_field_equals_continuous_run():
    """P9: step(5), get the field, set_init (same shell), step(6) == step(11)."""
    u0 = JI.hash_field(40, 40, 40, seed=2)
    with jb.Jacobi3D((40, 40, 40), (2, 2, 2)) as s:
        s.set_init(u0)
        s.step(5)
        mid = s.field(u0)
        s.set_init(mid)
        s.step(6)
        assert_bits(s.field(u0), ref(u0, 11))


def test_structured_fields_on_gpu():
    """P1 constant and P2 linear fields stay bit-identical on the GPU too."""
    for u0 in (JI.constant_field(30, 20, 10, 3.25), JI.linear_field(30, 20, 10)):
        assert_bits(run(u0, (3, 2, 2), 8), u0)


def test_ghost_conservation_p11():
    """After the exchange, every LOCAL ghost face equals the neighbour's boundary layer."""
    dims, blocks = (32, 24, 16), (2, 2, 2)
    u0 = JI.hash_field(*dims, seed=1)
    with jb.Jacobi3D(dims, blocks) as s:
        s.set_init(u0)
        s.step(3)
        ex, ey, ez = s.block_extent
        pads = {(x, y, z): s.block_padded(x, y, z) for x in range(2) for y in range(2) for z in range(2)}
        for (x, y, z), b in pads.items():
            if x == 0:
                assert_bits(b[1:-1, 1:-1, ex + 1], pads[(1, y, z)][1:-1, 1:-1, 1])
            if y == 0:
                assert_bits(b[1:-1, ey + 1, 1:-1], pads[(x, 1, z)][1:-1, 1, 1:-1])
            if z == 0:
                assert_bits(b[ez + 1, 1:-1, 1:-1], pads[(x, y, 1)][1, 1:-1, 1:-1])


def test_skip_exchange_is_wrong_and_flagged():
    """JAC_F_SKIP_EXCHANGE is timing-only: with ODF > 1 it must NOT match."""
    u0 = JI.hash_field(32, 32, 32, seed=1)
    got = run(u0, (2, 1, 1), 4, flags=J.JAC_F_SKIP_EXCHANGE)
    assert not np.array_equal(got, ref(u0, 4))


def test_c5_fine_grain_scaled():
    """C5's shape (32^3 blocks, 8 partitions) at 256^3: 512 blocks, 64 per partition."""
    u0 = JI.hash_field(256, 256, 256, seed=1)
    want = ref(u0, 12)
    assert_bits(run(u0, (8, 8, 8), 12, n_gpus=8, flags=J.JAC_F_VIRTUAL_GPUS), want)


def _lightcone_check(got, u0, n, corners, s=8):
    nz, ny, nx = (d - 2 for d in u0.shape)
    for (x0, y0, z0) in corners:
        lo = [max(0, c - n) for c in (z0, y0, x0)]
        hi = [min(N, c + s + n) for c, N in ((z0, nz), (y0, ny), (x0, nx))]
        sub = np.ascontiguousarray(u0[lo[0]:hi[0] + 2, lo[1]:hi[1] + 2, lo[2]:hi[2] + 2])
        res = ref(sub, n)
        a = res[z0 - lo[0] + 1:z0 - lo[0] + 1 + s, y0 - lo[1] + 1:y0 - lo[1] + 1 + s,
                x0 - lo[2] + 1:x0 - lo[2] + 1 + s]
        assert_bits(got[z0 + 1:z0 + 1 + s, y0 + 1:y0 + 1 + s, x0 + 1:x0 + 1 + s], a)


def test_c2_full_size_bench_config():
    """BASELINE.json configs[1] at full size in the bench's launch configuration
    (512^3, device hash init, 100 iterations): bit-hash identical across ODF 1, 8, 64,
    and light-cone sub-cubes at block seams / corners / centre equal the oracle."""
    nx = 512
    n = 100
    u0 = JI.hash_field(nx, nx, nx, seed=1)
    hashes = []
    got = None
    for blocks in [(2, 2, 2), (1, 1, 1), (4, 4, 4)]:
        with jb.Jacobi3D((nx, nx, nx), blocks) as s:
            s.set_init_hash(1)
            s.step(n)
            f = s.field(u0)
        hashes.append(oracle.bithash(f))
        if got is None:
            got = f
    assert len(set(hashes)) == 1
    _lightcone_check(got, u0, n, [(0, 0, 0), (252, 252, 252), (504, 100, 255), (127, 383, 504)])


@pytest.mark.parametrize("variant", ["0", "1", "3", "4", "5", "12", "13", "14", "15"])
@pytest.mark.parametrize("dims,blocks", [((64, 40, 36), (2, 2, 2)), ((128, 34, 20), (2, 1, 1)),
                                         ((58, 30, 17), (2, 1, 1)), ((130, 51, 33), (1, 3, 1))])
def test_tma_tile_variants(monkeypatch, variant, dims, blocks):
    """Every TMA tile variant (wide 64+halo, narrow 32+halo, exact 32, exact 64) on
    block widths 32, 64, 29 and 130, forced through JAC_VARIANT (ignored where the
    variant cannot cover the block row)."""
    monkeypatch.setenv("JAC_EXPERIMENT", "1")
    monkeypatch.setenv("JAC_VARIANT", variant)
    u0 = JI.hash_field(*dims, seed=3)
    assert_bits(run(u0, blocks, 5), ref(u0, 5))


@pytest.mark.parametrize("threads", [1, 3])
@pytest.mark.parametrize("dims,blocks,extra", [((64, 48, 40), (2, 3, 2), 0), ((96, 64, 64), (3, 2, 4), 0),
                                               ((64, 64, 64), (2, 2, 2), 1 << 5), ((40, 40, 40), (1, 1, 1), 0)])
def test_paper_style_per_block_mode(threads, dims, blocks, extra):
    """NEXT-2: per-block streams, per-face pack/unpack launches, event ordering,
    several launching host threads -- bit-identical to the oracle (and so to the
    batched path)."""
    u0 = JI.hash_field(*dims, seed=1)
    nz2, ny2, nx2 = u0.shape
    with jb.Jacobi3D(dims, blocks, flags=J.JAC_F_PER_BLOCK | extra) as s:
        s.set_option(J.JAC_OPT_LAUNCH_THREADS, threads)
        s.set_init(u0)
        s.step(3)
        s.step(4)
        got = s.field(u0)
        st = s.stats()
    assert_bits(got, ref(u0, 7))
    nb = blocks[0] * blocks[1] * blocks[2]
    assert st["kernels_per_iter"] == nb + 2 * st["local_faces"]


def test_autotune_picks_a_wide_variant_and_stays_exact():
    """jac_create times the 6- and 4-stage wide tiles on this GPU and keeps one;
    either way the result is the oracle's."""
    u0 = JI.hash_field(192, 96, 64, seed=2)
    with jb.Jacobi3D((192, 96, 64), (1, 1, 1)) as s:
        assert s.stats()["sweep_variant"] in (0, 5)
        s.set_init(u0)
        s.step(6)
        assert_bits(s.field(u0), ref(u0, 6))


@pytest.mark.parametrize("dense", [True, False])
@pytest.mark.parametrize("dims,blocks", [((64, 64, 64), (2, 2, 2)), ((70, 37, 23), (5, 1, 1)),
                                         ((96, 66, 40), (3, 3, 5)), ((33, 5, 9), (1, 1, 3))])
def test_get_block_every_block(monkeypatch, dense, dims, blocks):
    """jac_get_block (north-star call 4): every block's interior equals the oracle's
    slice [iz*ez:(iz+1)*ez, iy*ey:.., ix*ex:..] -- C1 and ragged decompositions, dense
    rows (ex % 8 == 0) and the padded layout."""
    if not dense:
        monkeypatch.setenv("JAC_EXPERIMENT", "1")
        monkeypatch.setenv("JAC_NO_DENSE", "1")
    u0 = JI.hash_field(*dims, seed=3)
    n = 6
    want = ref(u0, n)
    with jb.Jacobi3D(dims, blocks) as s:
        s.set_init(u0)
        s.step(n)
        ex, ey, ez = s.block_extent
        for iz in range(blocks[2]):
            for iy in range(blocks[1]):
                for ix in range(blocks[0]):
                    b = s.block(ix, iy, iz)
                    assert b.shape == (ez, ey, ex)
                    assert_bits(b, want[1 + iz * ez:1 + (iz + 1) * ez, 1 + iy * ey:1 + (iy + 1) * ey,
                                         1 + ix * ex:1 + (ix + 1) * ex])
        with pytest.raises(ValueError):  # the binding refuses a wrong-shaped buffer
            J.jac_get_block(s.ctx, 0, 0, 0, np.empty((ez, ey, ex + 1)))
        with pytest.raises(ValueError):
            J.jac_get_block(s.ctx, 0, 0, 0, np.empty((ez, ey, ex), dtype=np.float32))


@pytest.mark.parametrize("blocks", [(1, 1, 1), (2, 2, 2), (16, 16, 16)])
def test_ring_refill_race_regression(blocks):
    """Regression guard for the staging ring's write-after-read race:
    the first sweeps after init at 512^3, repeated, compared in full with the oracle.
    The racy ring showed stale 32-point row segments at n = 1 in most runs of a build
    whose scheduling delayed the first plane's loads (profiles/r02_ring_war_race.txt)."""
    nx = 512
    u0 = JI.hash_field(nx, nx, nx, seed=1)
    for n in (1, 2):
        want = ref(u0, n).view(np.uint64)
        for _ in range(2):
            with jb.Jacobi3D((nx, nx, nx), blocks) as s:
                s.set_init_hash(1)
                s.step(n)
                got = s.field(u0)
            bad = np.argwhere(got.view(np.uint64) != want)
            assert len(bad) == 0, f"n={n} blocks {blocks}: {len(bad)} stale values, first {bad[:3].tolist()}"
