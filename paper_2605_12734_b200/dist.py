"""One-process-per-GPU plumbing over torch.distributed (no data-path collective).

The only things that cross torch.distributed are the ranks' 256-byte IPC records
(all-gathered once at setup) and host barriers.  Faces then move by direct peer
stores from inside the sweep kernel over NVLink (include/jacobi3d.h,
jac_create_rank), synchronised by device flags -- the single-copy replacement of
the paper's two-copy IPC staging through a communication buffer.
"""
from __future__ import annotations

import os
from typing import List, Optional, Sequence

from .jacobi3d import (JAC_F_NCCL, Jacobi3D, jac_export_ipc, jac_import_ipc, jac_nccl_get_unique_id,
                       jac_nccl_init, jac_plan, jac_plan_face)


def exchange_records(record: bytes, world: int) -> List[bytes]:
    """All-gather one bytes record per rank (rank order)."""
    import torch.distributed as dist

    out: List[Optional[bytes]] = [None] * world
    dist.all_gather_object(out, record)
    return [bytes(r) for r in out]


def neighbor_ranks(dims, blocks, n_gpus, gpu_grid, rank) -> List[int]:
    """Face-adjacent ranks of ``rank`` from the host planner (jac_plan_face)."""
    g, _ = jac_plan(*dims, *blocks, n_gpus, gpu_grid)
    lb = [blocks[d] // g[d] for d in range(3)]
    px, py, pz = rank % g[0], (rank // g[0]) % g[1], rank // (g[0] * g[1])
    peers = set()
    for iz in range(pz * lb[2], (pz + 1) * lb[2]):
        for iy in range(py * lb[1], (py + 1) * lb[1]):
            for ix in range(px * lb[0], (px + 1) * lb[0]):
                if 0 < ix % lb[0] < lb[0] - 1 and 0 < iy % lb[1] < lb[1] - 1 and 0 < iz % lb[2] < lb[2] - 1:
                    continue  # interior block of the partition: no remote faces
                for f in range(6):
                    kind, owner = jac_plan_face(*dims, *blocks, n_gpus, gpu_grid, ix, iy, iz, f)
                    if kind == 2:
                        peers.add(owner)
    return sorted(peers)


def create_rank_context(dims: Sequence[int], blocks: Sequence[int], gpu_grid=None, flags: int = 0,
                        device: Optional[int] = None) -> Jacobi3D:
    """Collective: every rank of the default process group creates its partition's
    context, then the ranks swap IPC records and open their neighbours' memory."""
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", rank))
    J = Jacobi3D(dims, blocks, n_gpus=world, gpu_grid=gpu_grid, flags=flags, rank=rank, device=device)
    if flags & JAC_F_NCCL:  # ablation transport: NCCL communicator instead of IPC peer stores
        uid = jac_nccl_get_unique_id() if rank == 0 else b""
        uid = exchange_records(uid, world)[0]
        jac_nccl_init(J.ctx, uid)
    else:
        recs = exchange_records(jac_export_ipc(J.ctx), world)
        jac_import_ipc(J.ctx, recs)
    dist.barrier()
    return J


def destroy_rank_context(J: Jacobi3D) -> None:
    """Collective: no rank frees memory a neighbour may still store into."""
    import torch.distributed as dist

    dist.barrier()
    J.close()
    dist.barrier()
