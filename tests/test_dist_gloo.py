"""N>1 host-side logic on CPU with the gloo backend, world_size 2 (no GPU): the IPC
record exchange used by dist.create_rank_context, the neighbour-rank sets (must be
symmetric), and the bench's weak/strong workload geometry."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_12734_b200.dist import exchange_records, neighbor_ranks
    recs = exchange_records(bytes([rank]) * 256, world)
    dims, blocks = (64, 64, 128), (2, 2, 4)
    peers = neighbor_ranks(dims, blocks, world, None, rank)
    all_peers = [None] * world
    dist.all_gather_object(all_peers, peers)
    q.put((rank, [r[0] for r in recs], [len(r) for r in recs], all_peers))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_record_exchange_and_neighbours():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, firsts, lens, all_peers in out:
        assert firsts == [0, 1] and lens == [256, 256]
        assert all_peers == [[1], [0]]


@pytest.mark.parametrize("world,grid", [(2, (1, 1, 2)), (4, (1, 2, 2)), (8, (2, 2, 2))])
def test_neighbour_sets_symmetric(world, grid):
    from paper_2605_12734_b200.dist import neighbor_ranks
    dims, blocks = (128, 128, 128), (4, 4, 4)
    peers = {r: neighbor_ranks(dims, blocks, world, grid, r) for r in range(world)}
    for r, ps in peers.items():
        assert len(ps) == sum(1 for g in grid if g > 1)  # one face-neighbour per split dim (2 parts)
        for p in ps:
            assert r in peers[p]


def test_bench_geometry():
    import bench
    assert bench.blocks_for_odf((512, 512, 512), 16) == (2, 2, 4)
    assert bench.blocks_for_odf((768, 768, 768), 8) == (2, 2, 2)
    for n in (1, 2, 4, 8):
        dims, blocks, g, _, scaling = bench.workload("c2", n, 8)
        assert scaling == "weak" and dims[0] * dims[1] * dims[2] == n * 512 ** 3
        assert blocks[0] * blocks[1] * blocks[2] == 8 * n
        dims, blocks, g, _, scaling = bench.workload("c4", n, 16)
        assert scaling == "strong" and blocks[0] * blocks[1] * blocks[2] == 16 * n
    # C4 ODF 16 block shapes at 1/2/4/8 GPUs
    shapes = [tuple(1536 // b for b in bench.workload("c4", n, 16)[1]) for n in (1, 2, 4, 8)]
    assert shapes == [(768, 768, 384), (768, 384, 384), (384, 384, 384), (384, 384, 192)]
