"""Small driver for ncu captures of the sweep kernel (no graph: one launch per
iteration).  python tools/profile_sweep.py --dims 512 512 512 --blocks 2 2 2 --iters 4 [--flags F]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_12734_b200 as jb

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=3, default=[512, 512, 512])
ap.add_argument("--blocks", type=int, nargs=3, default=[2, 2, 2])
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--flags", type=int, default=0)
a = ap.parse_args()
with jb.Jacobi3D(tuple(a.dims), tuple(a.blocks), flags=a.flags) as s:
    s.set_init_hash(1)
    ms = s.profile_sweep(a.iters)
    print(f"dims={a.dims} blocks={a.blocks} flags={a.flags} avg sweep {ms*1e3:.1f} us "
          f"-> {16*a.dims[0]*a.dims[1]*a.dims[2]/(ms*1e-3)/1e9:.0f} GB/s algorithmic")
