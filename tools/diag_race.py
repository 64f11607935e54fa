"""Hunt for rare wrong values: run n sweeps (hash init) many times at a size / block
grid and compare the whole field with the oracle; report mismatch counts and, for each
failing run, where the wrong values sit relative to blocks, tiles (64 x 16) and
z-chunks (16 planes).  DIMS=768 BLOCKS=2x2x2 N=1 REPS=20 python tools/diag_race.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import jac_inputs as JI
import oracle
import paper_2605_12734_b200 as jb

nx = int(os.environ.get("DIMS", "768"))
blocks = tuple(int(v) for v in os.environ.get("BLOCKS", "2x2x2").split("x"))
ns = [int(v) for v in os.environ.get("N", "1").split(",")]
reps = int(os.environ.get("REPS", "20"))
u0 = JI.hash_field(nx, nx, nx, seed=1)
ex, ey, ez = (nx // b for b in blocks)
for n in ns:
    t0 = time.time()
    want = oracle.jacobi3d_omp(u0, n)[0]
    wv = want.view(np.uint64)
    print(f"oracle n={n} {time.time() - t0:.1f}s", flush=True)
    fails = 0
    for rep in range(reps):
        with jb.Jacobi3D((nx, nx, nx), blocks) as s:
            s.set_init_hash(1)
            s.step(n)
            got = s.field(u0)
            var = s.stats()["sweep_variant"]
        bad = np.argwhere(got.view(np.uint64) != wv)
        if len(bad) == 0:
            continue
        fails += 1
        z, y, x = (bad[:, 0] - 1), (bad[:, 1] - 1), (bad[:, 2] - 1)  # interior coords
        print(f"n={n} rep={rep} variant={var} mismatches={len(bad)} z[{z.min()},{z.max()}] y[{y.min()},{y.max()}] "
              f"x[{x.min()},{x.max()}]", flush=True)
        # runs: group by (z, y) rows
        rows = {}
        for zz, yy, xx in zip(z, y, x):
            rows.setdefault((int(zz), int(yy)), []).append(int(xx))
        for (zz, yy), xs in list(rows.items())[:12]:
            xs.sort()
            print(f"   row z={zz} (blk {zz // ez} local {zz % ez}, chunk-local {zz % ez % 16}) y={yy} (blk {yy // ey} "
                  f"local {yy % ey}, tile-row {yy % ey % 16}) x {xs[0]}..{xs[-1]} n={len(xs)} "
                  f"(blk-local {xs[0] % ex}..{xs[-1] % ex}, tile {xs[0] % ex // 64})", flush=True)
        print(f"   distinct rows {len(rows)}", flush=True)
    print(f"n={n}: {fails}/{reps} runs with mismatches", flush=True)
