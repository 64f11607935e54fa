"""Same-box A/B of two builds (JAC_LIB_A / JAC_LIB_B, '' = in-tree) on graph-replayed
us/iter, one subprocess per (build, case) so each loads its own library."""
import json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = os.environ.get("CASES", "512x512x512:1x1x1,512x512x512:2x2x2,512x512x512:2x2x4,512x512x512:4x4x4,"
                       "512x512x512:8x8x8,768x768x768:2x2x2,1536x1536x1536:1x1x1").split(",")
CHILD = r'''
import os, sys, json
sys.path.insert(0, sys.argv[1])
from paper_2605_12734_b200 import Jacobi3D
dims = tuple(int(x) for x in sys.argv[2].split("x")); blocks = tuple(int(x) for x in sys.argv[3].split("x"))
n = max(10, int(4e9 / (dims[0] * dims[1] * dims[2])))
with Jacobi3D(dims, blocks) as J:
    J.set_init_hash(1); J.step(10); J.step(n)
    print(json.dumps([J.last_step_ms() / n * 1e3, J.stats()["sweep_variant"]]))
'''
for rep in range(int(os.environ.get("REPS", 2))):
    for case in CASES:
        d, b = case.split(":")
        res = []
        for lib in (os.environ.get("JAC_LIB_A", ""), os.environ.get("JAC_LIB_B", "build/ab/lib_prev.so")):
            env = dict(os.environ)
            env.pop("JAC_LIB", None)
            if lib:
                env["JAC_LIB"] = lib
            out = subprocess.run([sys.executable, "-c", CHILD, ROOT, d, b], capture_output=True, text=True, env=env)
            res.append(json.loads(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else [float("nan"), -1])
        print(f"{d} blocks {b}: new {res[0][0]:.1f} (v{res[0][1]})  prev {res[1][0]:.1f} (v{res[1][1]})  "
              f"({res[0][0] / res[1][0] - 1:+.1%})", flush=True)
