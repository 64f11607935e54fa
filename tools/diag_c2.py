"""Diagnostic: 512^3 parity per ODF and iteration count (mismatch counts and first
locations) against the OpenMP oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import jac_inputs as JI
import oracle
import paper_2605_12734_b200 as jb

nx = int(os.environ.get("NX", "512"))
u0 = JI.hash_field(nx, nx, nx, seed=1)
for n in [int(v) for v in os.environ.get("ITERS", "1,2,10,11").split(",")]:
    want = oracle.jacobi3d_omp(u0, n)[0]
    for blocks in [(1, 1, 1), (2, 2, 2), (4, 4, 4)]:
        for init in ("hash", "host"):
            with jb.Jacobi3D((nx, nx, nx), blocks) as s:
                if init == "hash":
                    s.set_init_hash(1)
                else:
                    s.set_init(u0)
                s.step(n)
                f = s.field(u0)
                st = s.stats()
            bad = np.argwhere(f.view(np.uint64) != want.view(np.uint64))
            print(f"n={n} blocks={blocks} init={init} variant={st['sweep_variant']} mismatches={len(bad)} "
                  f"first={bad[:3].tolist()} last={bad[-2:].tolist()}", flush=True)
