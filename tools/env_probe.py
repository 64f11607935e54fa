"""Graph-replayed us/iter of a 512^3 decomposition for values of one environment knob
read at jac_create.  KNOB=JAC_ORDER_EXP VALUES=0,1,2 BLOCKS=2x2x2 [DIMS=512x512x512]."""
import os, sys
os.environ.setdefault("JAC_EXPERIMENT", "1")  # the library reads experiment knobs only with this set
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_12734_b200 import Jacobi3D

knob = os.environ.get("KNOB", "JAC_ORDER_EXP")
dims = tuple(int(x) for x in os.environ.get("DIMS", "512x512x512").split("x"))
n = int(os.environ.get("N", 200))
for rep in range(int(os.environ.get("REPS", 3))):
    for bs in os.environ.get("BLOCKS", "2x2x2").split(","):
        blocks = tuple(int(x) for x in bs.split("x"))
        out = []
        for v in os.environ.get("VALUES", "0,1,2").split(","):
            os.environ[knob] = v
            with Jacobi3D(dims, blocks) as J:
                J.set_init_hash(1)
                J.step(20)
                J.step(n)
                out.append(f"{knob}={v}: {J.last_step_ms() / n * 1e3:.1f}")
        print(f"blocks {blocks}: " + " | ".join(out), flush=True)
