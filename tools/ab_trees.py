"""Same-box A/B of two source trees (ROOT_A = this repo, ROOT_B = another checkout with
its own built libjacobi3d.so, e.g. _r1/), graph-replayed us/iter per case, one child
process per (tree, case) so each loads its own binding and library; interleaved
repetitions, median reported.
    ROOT_B=_r1 CASES=512x512x512:16x16x16 REPS=3 python tools/ab_trees.py
2-D cases: "2d131072x98304:2x1" (dims:blocks); AB_GPUS=N runs jac_create(n_gpus=N)."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ROOTS = [os.environ.get("ROOT_A", ROOT), os.environ.get("ROOT_B", os.path.join(ROOT, "_prev"))]
CASES = os.environ.get("CASES", "512x512x512:1x1x1,512x512x512:2x2x2,512x512x512:4x4x4,512x512x512:8x8x8,"
                       "512x512x512:16x16x16,1024x1024x1024:32x32x32").split(",")
CHILD = r'''
import os, sys, json, time
sys.path.insert(0, sys.argv[1])
from paper_2605_12734_b200 import Jacobi3D
from paper_2605_12734_b200 import Jacobi2D
ngpu = int(os.environ.get("AB_GPUS", "1"))
two_d = sys.argv[2].startswith("2d")
dims = tuple(int(x) for x in sys.argv[2].replace("2d", "").split("x")); blocks = tuple(int(x) for x in sys.argv[3].split("x"))
pts = 1
for d in dims: pts *= d
n = max(10, int(4e9 * ngpu / pts))
with (Jacobi2D(dims, blocks, n_gpus=ngpu) if two_d else Jacobi3D(dims, blocks, n_gpus=ngpu)) as J:
    J.set_init_hash(1); J.step(10); time.sleep(0.25); J.step(n)
    ms = J.last_step_ms() / n
    time.sleep(0.25)
    sw = J.profile_sweep(10)
    print(json.dumps([ms * 1e3, sw * 1e3]))
'''
res = {c: [[], []] for c in CASES}
for rep in range(int(os.environ.get("REPS", 3))):
    for case in CASES:
        d, b = case.split(":")
        for k, root in enumerate(ROOTS):
            env = {k2: v for k2, v in os.environ.items() if k2 != "JAC_LIB"}
            out = subprocess.run([sys.executable, "-c", CHILD, root, d, b], capture_output=True, text=True, env=env)
            if out.returncode == 0:
                res[case][k].append(json.loads(out.stdout.strip().splitlines()[-1]))
            else:
                print(out.stderr[-800:], file=sys.stderr)
for case in CASES:
    a, b = res[case]
    if not a or not b:
        print(case, "FAILED")
        continue
    ma, mb = statistics.median(x[0] for x in a), statistics.median(x[0] for x in b)
    sa, sb = statistics.median(x[1] for x in a), statistics.median(x[1] for x in b)
    print(f"{case:28s} A {ma:8.1f} us/iter (sweep {sa:7.1f})  B {mb:8.1f} (sweep {sb:7.1f})  A/B {ma / mb - 1:+.2%}",
          flush=True)
