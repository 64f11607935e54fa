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
    ap.add_argument("--two-d", action="store_true", help="Jacobi2D (dims X Y 1, blocks BX BY 1)")
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    dims = tuple(a.dims)
    flags = a.flags | ((1 << 9) if a.two_d else 0)
    J = create_rank_context(dims, tuple(a.blocks), gpu_grid=a.grid, flags=flags, device=local)
    origin, extent = J.local_box()
    if a.two_d:  # 2-D padded index p = j*(nx+2) + i: the (nz+2)-plane formula with plane 0
        full2d = JI.hash_field2d(dims[0], dims[1], seed=2)
        box = np.ascontiguousarray(full2d[origin[1]:origin[1] + extent[1], origin[0]:origin[0] + extent[0]])[None]
    else:
        box = JI.hash_box(*dims, origin, extent, seed=2)
    if a.hash_init:
        J.set_init_hash(2)
    elif a.two_d:
        J.set_init_box(box, origin)
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
        if a.two_d:
            u0 = JI.hash_field2d(dims[0], dims[1], seed=2)
            want, _ = oracle.jacobi2d_omp(u0, a.iters)
            got = u0.copy()
            for (o, b, _) in parts:
                ox, oy, _ = o
                _, sy, sx = b.shape
                got[oy + 1:oy + sy - 1, ox + 1:ox + sx - 1] = b[0, 1:-1, 1:-1]
        else:
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
