"""Diagnostic: 512^3 ODF 1 parity, n=1 and n=3, repeated, mismatch counts."""
import os
import sys

root = os.environ.get("DIAG_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, root)
import numpy as np

import jac_inputs as JI
import oracle
import paper_2605_12734_b200 as jb

nx = 512
u0 = JI.hash_field(nx, nx, nx, seed=1)
tag = os.environ.get("TAG", "")
for n in (1, 3):
    want = oracle.jacobi3d_omp(u0, n)[0]
    res = []
    for rep in range(4):
        with jb.Jacobi3D((nx, nx, nx), (1, 1, 1)) as s:
            s.set_init(u0)
            s.step(n)
            f = s.field(u0)
        res.append(int(np.count_nonzero(f.view(np.uint64) != want.view(np.uint64))))
    print(f"{tag} n={n} mismatches per run={res}", flush=True)
