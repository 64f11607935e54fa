"""Multi-GPU parity (one process per GPU, IPC peer stores + device-flag barrier),
bit-exact against the oracle.  Needs >= 2 GPUs (gpurun --gpus 2 / 4); skipped on a
1-GPU box, where the partition logic is covered by JAC_F_VIRTUAL_GPUS tests."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _ngpu():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


CASES = [
    # (nproc, dims, blocks, grid, iters, flags, hash)
    (2, (64, 48, 80), (2, 2, 4), None, 21, 0, False),          # 1x1x2 split, ODF 8
    (2, (70, 37, 46), (2, 1, 2), None, 7, 0, False),           # ragged, odd x extent
    (2, (64, 64, 64), (2, 2, 2), (2, 1, 1), 9, 0, True),       # x split: strided remote x-faces
    (2, (48, 48, 48), (2, 2, 2), None, 11, 1 << 4, False),     # unfused pack + ghost kernel, remote pull
    (2, (48, 48, 48), (2, 2, 2), None, 5, 1 << 1, False),      # no graph
    (4, (64, 64, 64), (2, 2, 4), None, 13, 0, False),          # 1x2x2
    (4, (64, 64, 64), (4, 2, 2), (2, 2, 1), 6, 1 << 5, False), # no TMA
    (8, (64, 64, 64), (4, 4, 4), None, 17, 0, False),          # 2x2x2, ODF 8
    (2, (256, 192, 1), (2, 4, 1), None, 13, 1 << 9, False),    # Jacobi2D, y split
    (4, (256, 192, 1), (4, 4, 1), None, 9, 1 << 9, True),      # Jacobi2D, 2x2 GPUs, hash init
    (2, (64, 48, 80), (2, 2, 4), None, 21, 1 << 2, False),     # NCCL transport ablation
    (4, (64, 64, 64), (4, 2, 2), (2, 2, 1), 7, 1 << 2, False), # NCCL, x-split (x-ghost layout)
    (2, (256, 192, 1), (2, 4, 1), None, 5, (1 << 2) | (1 << 9), False),  # NCCL + Jacobi2D
    # 128-wide blocks split in x: lean-path tiles (full, no y-face rows) whose x-edge
    # lanes store remote x faces through IPC pointers / into NCCL send buffers
    (2, (256, 64, 48), (2, 1, 1), (2, 1, 1), 9, 0, True),
    (2, (256, 64, 48), (2, 1, 1), (2, 1, 1), 9, 1 << 2, True),
    (4, (256, 128, 48), (2, 2, 1), (2, 2, 1), 7, 0, True),
    (2, (512, 96, 1), (2, 1, 1), (2, 1, 1), 9, 1 << 9, True),   # Jacobi2D lean tiles, x split
]


@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}_{c[2]}_{c[5]}" for c in CASES])
def test_multi_process_parity(case):
    n, dims, blocks, grid, iters, flags, hashed = case
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    import socket
    for attempt in range(4):  # a probed-free port can be taken before torchrun binds it
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--master-addr", "127.0.0.1",
               "--master-port", str(port), "--nproc-per-node", str(n),
               os.path.join(ROOT, "tools", "mp_parity.py"), "--dims", *map(str, dims), "--blocks", *map(str, blocks),
               "--iters", str(iters), "--flags", str(flags)]
        if grid:
            cmd += ["--grid", *map(str, grid)]
        if hashed:
            cmd += ["--hash-init"]
        if flags & (1 << 9):
            cmd += ["--two-d"]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
        if r.returncode == 0 or "EADDRINUSE" not in r.stderr:
            break
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout


# ---------------------------------------------------------------- single process, N GPUs
# jac_create(n_gpus > 1): one process drives every GPU; the
# sub-contexts run the rank path with plain peer pointers.
SP_CASES = [
    # (n_gpus, dims, blocks, grid, iters, flags, hash)
    (2, (64, 48, 80), (2, 2, 4), None, 21, 0, False),         # 1x1x2, ODF 8
    (2, (128, 40, 36), (2, 1, 1), (2, 1, 1), 9, 0, True),     # x split: remote x-ghost arrays
    (2, (96, 40, 36), (2, 1, 1), (2, 1, 1), 7, 0, False),     # x split, host init: pitched staging rows
    (2, (48, 64, 40), (1, 2, 1), (1, 2, 1), 5, 0, False),     # y split, host init: one run per plane
    (2, (48, 48, 48), (2, 2, 2), None, 11, 1 << 4, False),    # unfused pack + barrier + pull
    (2, (48, 48, 48), (2, 2, 2), None, 5, 1 << 1, False),     # no graph (interleaved launches)
    (2, (64, 64, 64), (2, 2, 2), None, 6, 1 << 5, False),     # plain-load sweep + barrier
    (4, (64, 64, 64), (2, 2, 4), None, 13, 0, False),         # 1x2x2
    (4, (256, 128, 48), (2, 2, 1), (2, 2, 1), 7, 0, True),    # lean tiles, x and y splits
    (8, (64, 64, 64), (4, 4, 4), None, 17, 0, False),         # 2x2x2
]


@pytest.mark.parametrize("case", SP_CASES, ids=[f"sp_n{c[0]}_{c[2]}_{c[5]}" for c in SP_CASES])
def test_single_process_multi_gpu_parity(case):
    import numpy as np

    sys.path.insert(0, ROOT)
    import jac_inputs as JI
    import oracle
    import paper_2605_12734_b200 as jb

    n, dims, blocks, grid, iters, flags, hashed = case
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    u0 = JI.hash_field(*dims, seed=2)
    with jb.Jacobi3D(dims, blocks, n_gpus=n, gpu_grid=grid, flags=flags) as s:
        if hashed:
            s.set_init_hash(2)
        else:
            s.set_init(u0)
        for k in (3, 1, iters - 4):
            s.step(k)
        got = s.field(u0)
        st = s.stats()
        s_grid = s.gpu_grid
        blk = s.block(blocks[0] - 1, blocks[1] - 1, blocks[2] - 1)  # owned by the last device
    want = oracle.jacobi3d_omp(u0, iters)[0]
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    ex, ey, ez = (dims[d] // blocks[d] for d in range(3))
    assert np.array_equal(blk, want[-ez - 1:-1, -ey - 1:-1, -ex - 1:-1])
    assert st["partitions"] == n and st["remote_faces"] > 0
    if flags == 0:  # init: 2 barriers; each of the 3 jac_step calls: `diameter` aligning
        # barrier rounds; 1 signal per sweep
        g = s_grid
        diameter = (g[0] - 1) + (g[1] - 1) + (g[2] - 1)
        assert st["fused_sync"] == 1 and st["epoch_min"] == st["epoch_max"] == 2 + 3 * diameter + iters


def test_single_process_multi_gpu_2d():
    import numpy as np

    sys.path.insert(0, ROOT)
    import jac_inputs as JI
    import oracle
    import paper_2605_12734_b200 as jb

    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    u0 = JI.hash_field2d(256, 192, seed=1)
    with jb.Jacobi2D((256, 192), (2, 4), n_gpus=2) as s:
        s.set_init(u0)
        s.step(13)
        got = s.field(u0)
    assert np.array_equal(got.view(np.uint64), oracle.jacobi2d_omp(u0, 13)[0].view(np.uint64))


def test_single_process_multi_gpu_api_surface():
    """The group context answers the whole C ABI like a 1-GPU one: layout, owner,
    regions spanning devices, padded blocks, stats totals, options, errors naming the
    argument, and the watchdog option on every device."""
    import numpy as np

    sys.path.insert(0, ROOT)
    import jac_inputs as JI
    import oracle
    import paper_2605_12734_b200 as jb
    from paper_2605_12734_b200 import jacobi3d as J

    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    dims, blocks = (64, 48, 80), (2, 2, 4)
    u0 = JI.hash_field(*dims, seed=5)
    want = oracle.jacobi3d_omp(u0, 7)[0]
    with jb.Jacobi3D(dims, blocks, n_gpus=2) as s:
        assert s.gpu_grid == (1, 1, 2)
        assert s.owner(0, 0, 0) == 0 and s.owner(1, 1, 3) == 1
        o, e = s.local_box()
        assert o == (0, 0, 0) and e == (66, 50, 82)
        s.set_option(J.JAC_OPT_WATCHDOG_MS, 30000)
        s.set_init(u0)
        s.step(7)
        # a region across the device seam (z = 40)
        reg = s.region((5, 3, 30), (20, 30, 20))
        assert np.array_equal(reg, want[31:51, 4:34, 6:26])
        pb = s.block_padded(1, 1, 2)   # device 1, ghosts written by device 0 over NVLink
        ex, ey, ez = s.block_extent
        assert np.array_equal(pb[1:-1, 1:-1, 1:-1], want[1 + 2 * ez:1 + 3 * ez, 1 + ey:1 + 2 * ey, 1 + ex:1 + 2 * ex])
        assert np.array_equal(pb[0, 1:-1, 1:-1], want[2 * ez, 1 + ey:1 + 2 * ey, 1 + ex:1 + 2 * ex])  # z- ghost
        st = s.stats()
        assert st["local_blocks"] == 16 and st["partitions"] == 2 and st["kernels_per_iter"] == 1
        assert s.iterations == 7 and s.last_step_ms() > 0
        with pytest.raises(J.JacError) as ei:
            s.block(2, 0, 0)
        assert ei.value.code == J.JAC_EINVAL
        with pytest.raises(J.JacError) as ei:
            J.jac_export_ipc(s.ctx)
        assert ei.value.code == J.JAC_ESTATE
    with pytest.raises(J.JacError) as ei:
        jb.Jacobi3D(dims, blocks, n_gpus=2, flags=J.JAC_F_NCCL)
    assert ei.value.code == J.JAC_EINVAL


def test_single_process_multi_gpu_watchdog(monkeypatch):
    """Real GPUs, one process: partitions that never signal make their neighbours'
    waits give up after the watchdog limit; jac_step reports it (JAC_ECUDA "peer
    watchdog") instead of hanging, and the devices stay usable."""
    import numpy as np

    sys.path.insert(0, ROOT)
    import jac_inputs as JI
    import oracle
    import paper_2605_12734_b200 as jb
    from paper_2605_12734_b200 import jacobi3d as J

    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    dims, blocks = (64, 48, 80), (2, 2, 4)
    u0 = JI.hash_field(*dims, seed=1)
    monkeypatch.setenv("JAC_EXPERIMENT", "1")
    monkeypatch.setenv("JAC_HOLD_SIGNAL", "1")
    with jb.Jacobi3D(dims, blocks, n_gpus=2) as s:
        s.set_option(J.JAC_OPT_WATCHDOG_MS, 300)
        s.set_init(u0)
        with pytest.raises(J.JacError) as ei:
            s.step(4)
        assert ei.value.code == J.JAC_ECUDA and "watchdog" in str(ei.value)
    monkeypatch.delenv("JAC_HOLD_SIGNAL")
    monkeypatch.delenv("JAC_EXPERIMENT")
    with jb.Jacobi3D(dims, blocks, n_gpus=2) as s:
        s.set_init(u0)
        s.step(4)
        assert np.array_equal(s.field(u0).view(np.uint64), oracle.jacobi3d_omp(u0, 4)[0].view(np.uint64))
