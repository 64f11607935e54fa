"""Inter-partition exchange on ONE GPU: JAC_F_VIRTUAL_GPUS
hosts every partition of an n_gpus decomposition on device 0 and sweeps them with one
kernel per iteration, but the faces between partitions take the REMOTE path of a
multi-GPU run -- per-partition remote masks, the remote-first item order, the
per-partition epoch / flag / count words with the in-sweep wait (wait_peers) and
signal (signal_done), the barrier kernel, and, with JAC_F_NCCL, the packed send /
receive buffers of the NCCL transport moved by an on-device copy kernel.

The paper's transport layer: intra-node inter-process transfers (§4.1
item 2) and transport selection by placement.  Every case is bit-exact
against the undecomposed CPU oracle (reading R15), and the epoch
counters prove the handshake ran once per sweep.  Kernels that wait on one another
never share a GPU (B200_PROFILING.md): inside one kernel the previous sweep has
completed, so the waits check the bookkeeping, not timing."""
from __future__ import annotations

import numpy as np
import pytest

import jac_inputs as JI
import oracle
import paper_2605_12734_b200 as jb
from paper_2605_12734_b200 import jacobi3d as J

pytestmark = pytest.mark.gpu

V = J.JAC_F_VIRTUAL_GPUS


def bits(a, b):
    assert a.shape == b.shape
    bad = np.flatnonzero(a.view(np.uint64) != b.view(np.uint64))
    assert bad.size == 0, f"{bad.size} mismatches, first at {np.unravel_index(bad[0], a.shape)}"


# (gpu grid, dims, global blocks): remote faces in z only, y+z, x only (strided x-ghost
# arrays), and all three directions (the 8-GPU decomposition of C3x8 / C4x8 / C5)
GRIDS = [
    ((1, 1, 2), (64, 48, 80), (2, 2, 4)),
    ((1, 2, 2), (64, 64, 64), (2, 2, 4)),
    ((2, 1, 1), (128, 40, 36), (2, 1, 1)),
    ((2, 2, 2), (64, 64, 64), (4, 4, 4)),
    ((2, 2, 2), (96, 64, 66), (2, 2, 2)),   # one 48x32x33 block per partition, ragged tiles
]
MODES = {"fused": V, "nccl_layout": V | J.JAC_F_NCCL, "unfused": V | J.JAC_F_UNFUSED_PACK,
         "plain_barrier": V | J.JAC_F_NO_TMA}


def run_virtual(dims, blocks, grid, flags, n, seed=2, steps=None, hashed=False):
    ng = grid[0] * grid[1] * grid[2]
    u0 = JI.hash_field(*dims, seed=seed)
    with jb.Jacobi3D(dims, blocks, n_gpus=ng, gpu_grid=grid, flags=flags) as s:
        if hashed:
            s.set_init_hash(seed)
        else:
            s.set_init(u0)
        st0 = s.stats()
        for k in (steps or [n]):
            s.step(k)
        return u0, s.field(u0), st0, s.stats()


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("grid,dims,blocks", GRIDS, ids=["x".join(map(str, g[0])) + f"_{g[2]}" for g in GRIDS])
def test_virtual_remote_bit_exact(grid, dims, blocks, mode):
    n = 13
    u0, got, st0, st = run_virtual(dims, blocks, grid, MODES[mode], n, steps=[3, 10])
    bits(got, oracle.jacobi3d_omp(u0, n)[0])
    ng = grid[0] * grid[1] * grid[2]
    assert st["partitions"] == ng
    assert st["remote_faces"] > 0
    if mode == "fused":
        # the sweep carries the ordering: one kernel per iteration, remote items first,
        # and every partition's epoch advanced by exactly one per sweep
        assert st["fused_sync"] == 1 and st["kernels_per_iter"] == 1
        assert 0 < st["remote_items"]
        assert st["epoch_min"] == st["epoch_max"] == st0["epoch_max"] + n
    elif mode == "nccl_layout":
        assert st["fused_sync"] == 0 and st["kernels_per_iter"] == 3  # sweep + copy + unpack
    elif mode in ("unfused", "plain_barrier"):
        # barrier kernels between the phases: each partition signals once per barrier
        per_iter = 2 if mode == "unfused" else 1
        assert st["epoch_min"] == st["epoch_max"] == st0["epoch_max"] + per_iter * n


def test_virtual_remote_init_epochs():
    """set_init runs two barriers (before the copy, after it): epochs 0 -> 2."""
    _, _, st0, _ = run_virtual((64, 64, 64), (2, 2, 2), (2, 2, 2), V, 0)
    assert st0["epoch_min"] == st0["epoch_max"] == 2


@pytest.mark.parametrize("flags", [V, V | J.JAC_F_NCCL])
def test_virtual_remote_hash_init_and_graph_boundaries(flags):
    """Device hash init, 25 iterations across the 10-iteration graph boundary, and a
    non-graph run: all bit-exact on the 2x2x2 grid."""
    dims, blocks, grid = (64, 64, 64), (2, 2, 4), (2, 2, 2)
    u0, got, _, _ = run_virtual(dims, blocks, grid, flags, 25, seed=3, steps=[1, 10, 14], hashed=True)
    bits(got, oracle.jacobi3d_omp(u0, 25)[0])
    u0, got, _, _ = run_virtual(dims, blocks, grid, flags | J.JAC_F_NO_GRAPH, 7, seed=3)
    bits(got, oracle.jacobi3d_omp(u0, 7)[0])


@pytest.mark.parametrize("flags", [V, V | J.JAC_F_NCCL])
@pytest.mark.parametrize("grid,blocks", [((1, 2, 1), (2, 4, 1)), ((2, 2, 1), (4, 4, 1)), ((2, 1, 1), (2, 1, 1))])
def test_virtual_remote_2d(grid, blocks, flags):
    """Jacobi2D (NEXT-1) through the same remote path (x-split: strided x faces)."""
    dims = (256, 192)
    u0 = JI.hash_field2d(*dims, seed=1)
    with jb.Jacobi2D(dims, blocks[:2], n_gpus=grid[0] * grid[1], gpu_grid=grid[:2], flags=flags) as s:
        s.set_init(u0)
        s.step(4)
        s.step(9)
        got = s.field(u0)
        st = s.stats()
    bits(got, oracle.jacobi2d_omp(u0, 13)[0])
    assert st["remote_faces"] > 0


def test_virtual_remote_lean_x_split():
    """128-wide blocks split in x: lean-path tiles whose x-edge lanes store remote x
    faces (the x-ghost arrays of another partition) or pack them (NCCL layout)."""
    dims, blocks, grid = (256, 64, 48), (2, 1, 1), (2, 1, 1)
    for flags in (V, V | J.JAC_F_NCCL):
        u0, got, _, _ = run_virtual(dims, blocks, grid, flags, 9)
        bits(got, oracle.jacobi3d_omp(u0, 9)[0])


def test_negative_control_dropped_remote_stores(monkeypatch):
    """With the remote stores disabled (experiment knob) the result must differ from
    the oracle -- the remote path, not a local shortcut, carries the faces."""
    monkeypatch.setenv("JAC_EXPERIMENT", "1")
    monkeypatch.setenv("JAC_DROP_REMOTE", "1")
    for flags in (V, V | J.JAC_F_NCCL):
        u0, got, _, st = run_virtual((64, 64, 64), (2, 2, 2), (2, 2, 2), flags, 5)
        assert st["experiment"] != 0
        want = oracle.jacobi3d_omp(u0, 5)[0]
        assert not np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_watchdog_reports_instead_of_trapping(monkeypatch):
    """A partition that never signals: its neighbours' waits give up after the
    watchdog limit, jac_step returns JAC_ECUDA ("peer watchdog"), and the CUDA context
    stays usable (a new context afterwards is bit-exact)."""
    monkeypatch.setenv("JAC_EXPERIMENT", "1")
    monkeypatch.setenv("JAC_HOLD_SIGNAL", "1")
    dims, blocks, grid = (64, 64, 64), (2, 2, 2), (1, 1, 2)
    u0 = JI.hash_field(*dims, seed=1)
    with jb.Jacobi3D(dims, blocks, n_gpus=2, gpu_grid=grid, flags=V) as s:
        s.set_option(J.JAC_OPT_WATCHDOG_MS, 200)
        s.set_init(u0)
        with pytest.raises(J.JacError) as ei:
            s.step(3)
        assert ei.value.code == J.JAC_ECUDA and "watchdog" in str(ei.value)
        s.field(u0)  # the device is still answering
    monkeypatch.delenv("JAC_HOLD_SIGNAL")
    monkeypatch.delenv("JAC_EXPERIMENT")
    _, got, _, _ = run_virtual(dims, blocks, grid, V, 4, seed=1)
    bits(got, oracle.jacobi3d_omp(u0, 4)[0])


def test_fuzz_virtual_remote():
    """Seeded random shapes / grids / modes through the remote path (16 cases)."""
    rng = np.random.default_rng(4242)
    done = 0
    while done < 16:
        b = [int(rng.choice([1, 2, 2, 4])) for _ in range(3)]
        e = [int(rng.choice([3, 8, 17, 32, 33, 64, 65])) for _ in range(3)]
        dims = tuple(b[d] * e[d] for d in range(3))
        if dims[0] * dims[1] * dims[2] > 1_200_000:
            continue
        grids = [g for g in [(1, 1, 2), (1, 2, 1), (2, 1, 1), (1, 2, 2), (2, 2, 1), (2, 1, 2), (2, 2, 2)]
                 if all(b[d] % g[d] == 0 for d in range(3))]
        if not grids:
            continue
        grid = grids[int(rng.integers(0, len(grids)))]
        flags = [V, V | J.JAC_F_NCCL, V | J.JAC_F_UNFUSED_PACK, V | J.JAC_F_NO_GRAPH][int(rng.integers(0, 4))]
        n = int(rng.integers(1, 12))
        u0, got, _, _ = run_virtual(dims, tuple(b), grid, flags, n, seed=1 + done % 3)
        want = oracle.jacobi3d_omp(u0, n)[0]
        bad = int(np.count_nonzero(got.view(np.uint64) != want.view(np.uint64)))
        assert bad == 0, f"dims {dims} blocks {b} grid {grid} flags {flags:#x} n {n}: {bad} mismatches"
        done += 1
