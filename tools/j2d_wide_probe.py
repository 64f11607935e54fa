"""Jacobi2D: per-point cost of very wide blocks vs the same points in 32768-wide rows or
blocks.  Each case: graph-replayed us/iter (median of R), then one profile_sweep launch
(the one an ncu capture with -k regex:sweep2d sees).  CASES='131072x4096,32768x16384,65536x8192:2x1'"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_12734_b200 import Jacobi2D

R = int(os.environ.get("R", "3"))
VARS = os.environ.get("VARS", "")  # forced tile variants (JAC_VARIANT), e.g. "5,15,1"
runs = [(c, v) for v in (VARS.split(",") if VARS else [None])
        for c in os.environ.get("CASES", "131072x4096,32768x16384,65536x8192:2x1").split(",")]
if VARS:
    os.environ["JAC_EXPERIMENT"] = "1"
for c, v in runs:
    if v is not None:
        os.environ["JAC_VARIANT"] = v
    d, _, b = c.partition(":")
    dims = tuple(map(int, d.split("x")))
    blocks = tuple(map(int, b.split("x"))) if b else (1, 1)
    with Jacobi2D(dims, blocks) as J:
        J.set_init_hash(1)
        if os.environ.get("NO_TIMING") != "1":
            J.step(10)
            n = max(10, int(4e9 / (dims[0] * dims[1])))
            t = []
            for _ in range(R):
                J.step(n)
                t.append(J.last_step_ms() / n * 1e3)
            us = statistics.median(t)
            print(f"{c}{'' if v is None else ' variant ' + v}: {us:.1f} us/iter, {us * 1e3 / (dims[0] * dims[1]):.4f} ns/point", flush=True)
        J.profile_sweep(1)
