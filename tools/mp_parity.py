"""Multi-process (one process per GPU) parity check, launched by torchrun.

    torchrun --standalone --nproc-per-node N tools/mp_parity.py --dims X Y Z --blocks BX BY BZ --iters I

Every rank owns one partition (jac_create_rank), swaps IPC records, initialises its
box from the shared input generator, runs the iterations (in uneven chunks, to cross
graph-unroll boundaries), reads its box back; rank 0 assembles the global field and
compares it bit for bit with the CPU oracle.  Exit code 0 = bit-exact.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch
import torch.distributed as dist

import jac_inputs as JI
from paper_2605_12734_b200.dist import create_rank_context, destroy_rank_context


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs=3, required=True)
    ap.add_argument("--blocks", type=int, nargs=3, required=True)
    ap.add_argument("--grid", type=int, nargs=3, default=None)
    ap.add_argument("--iters", type=int, default=9)
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--hash-init", action="store_true")
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    dims = tuple(a.dims)
    J = create_rank_context(dims, tuple(a.blocks), gpu_grid=a.grid, flags=a.flags, device=local)
    origin, extent = J.local_box()
    box = JI.hash_box(*dims, origin, extent, seed=2)
    if a.hash_init:
        J.set_init_hash(2)
    else:
        J.set_init_box(box, origin)
    chunks, left = [], a.iters
    for c in (3, 1, 12, 2):
        c = min(c, left)
        chunks.append(c)
        left -= c
    if left:
        chunks.append(left)
    for c in chunks:
        J.step(c)
    out = J.field_box(box.copy(), origin)
    st = J.stats()
    parts = [None] * world
    dist.all_gather_object(parts, (origin, out, st))
    ok = True
    if rank == 0:
        import oracle
        u0 = JI.hash_field(*dims, seed=2)
        want, _ = oracle.jacobi3d_omp(u0, a.iters)
        got = u0.copy()
        for (o, b, _) in parts:
            ox, oy, oz = o
            sz, sy, sx = b.shape
            # interiors only: the box's outer ring is ghost/shell
            got[oz + 1:oz + sz - 1, oy + 1:oy + sy - 1, ox + 1:ox + sx - 1] = b[1:-1, 1:-1, 1:-1]
        ok = np.array_equal(got.view(np.uint64), want.view(np.uint64))
        nbad = int(np.count_nonzero(got.view(np.uint64) != want.view(np.uint64)))
        print(f"MP_PARITY world={world} dims={dims} blocks={tuple(a.blocks)} iters={a.iters} "
              f"flags={a.flags} {'OK' if ok else 'FAIL'} mismatches={nbad} stats={[p[2] for p in parts]}",
              flush=True)
    flag = torch.tensor([0 if ok else 1], device="cuda")
    dist.broadcast(flag, 0)
    destroy_rank_context(J)
    dist.destroy_process_group()
    sys.exit(int(flag.item()))


if __name__ == "__main__":
    main()
