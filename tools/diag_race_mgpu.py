"""Soak test of the cross-GPU protocol (one process, jac_create(n_gpus=N), fused peer
stores + flag handshake): BOX^3 per GPU at ODF 8 (weak layout), n sweeps, REPS runs
each, full-field compare with the oracle.  N=4 BOX=256 N_IT=1,2,5 REPS=10."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import jac_inputs as JI
import oracle
import paper_2605_12734_b200 as jb

N = int(os.environ.get("N", "4"))
box = int(os.environ.get("BOX", "256"))
g = bench.weak_gpu_grid(N)
lb = bench.blocks_for_odf((box, box, box), int(os.environ.get("ODF", "8")))
dims = tuple(box * g[d] for d in range(3))
blocks = tuple(lb[d] * g[d] for d in range(3))
u0 = JI.hash_field(*dims, seed=1)
reps = int(os.environ.get("REPS", "10"))
flags = int(os.environ.get("FLAGS", "0"))
for n in [int(v) for v in os.environ.get("N_IT", "1,2,5").split(",")]:
    want = oracle.jacobi3d_omp(u0, n)[0].view(np.uint64)
    fails = []
    for rep in range(reps):
        with jb.Jacobi3D(dims, blocks, n_gpus=N, gpu_grid=g, flags=flags) as s:
            s.set_init_hash(1)
            s.step(n)
            got = s.field(u0)
        bad = np.argwhere(got.view(np.uint64) != want)
        if len(bad):
            fails.append((rep, len(bad), bad.min(axis=0).tolist(), bad.max(axis=0).tolist()))
    print(f"N={N} dims={dims} blocks={blocks} flags={flags} n={n}: {len(fails)}/{reps} runs with mismatches {fails[:3]}",
          flush=True)
