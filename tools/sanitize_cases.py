"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
each runs a few iterations through the C ABI and checks the oracle, so a sanitizer
run also proves the path it watched was the real one.
    compute-sanitizer --tool memcheck python tools/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import jac_inputs as JI
import oracle
import paper_2605_12734_b200 as jb
from paper_2605_12734_b200 import jacobi3d as J

V = J.JAC_F_VIRTUAL_GPUS
CASES = [
    ("c1_64cubed_odf8", (64, 64, 64), (2, 2, 2), 1, 0),
    ("blocks32_128cubed", (128, 128, 128), (4, 4, 4), 1, 0),
    ("ragged_70x37x23", (70, 37, 23), (2, 1, 1), 1, 0),
    ("unfused_pack", (64, 48, 40), (2, 3, 2), 1, J.JAC_F_UNFUSED_PACK),
    ("no_tma", (64, 48, 40), (2, 3, 2), 1, J.JAC_F_NO_TMA),
    ("per_block", (64, 48, 40), (2, 3, 2), 1, J.JAC_F_PER_BLOCK),
    ("virtual_remote_2x2x2", (64, 64, 64), (4, 4, 4), 8, V),
    ("virtual_remote_nccl_layout", (64, 64, 64), (2, 2, 4), 8, V | J.JAC_F_NCCL),
    ("virtual_remote_unfused", (48, 48, 48), (2, 2, 2), 2, V | J.JAC_F_UNFUSED_PACK),
]
only = set(sys.argv[1:])
fails = 0
for name, dims, blocks, ng, flags in CASES:
    if only and name not in only:
        continue
    u0 = JI.hash_field(*dims, seed=1)
    n = 3
    with jb.Jacobi3D(dims, blocks, n_gpus=ng, flags=flags) as s:
        s.set_init(u0)
        s.step(1)
        s.step(n - 1)
        got = s.field(u0)
    ok = np.array_equal(got.view(np.uint64), oracle.jacobi3d(u0, n).view(np.uint64))
    fails += not ok
    print(f"{name}: {'bit-exact' if ok else 'MISMATCH'}", flush=True)
u0 = JI.hash_field2d(96, 64, seed=1)
with jb.Jacobi2D((96, 64), (2, 2), n_gpus=4, flags=V) as s:
    s.set_init(u0)
    s.step(3)
    ok = np.array_equal(s.field(u0).view(np.uint64), oracle.jacobi2d(u0, 3).view(np.uint64))
    fails += not ok
    print(f"j2d_virtual_remote: {'bit-exact' if ok else 'MISMATCH'}", flush=True)
sys.exit(1 if fails else 0)
