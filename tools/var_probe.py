"""Graph-replayed us/iter per forced tile variant (JAC_VARIANT) for given block grids
of a 512^3 domain.  VARS='3,13' BLOCKS='16x16x16,8x8x8'."""
import os, sys
os.environ.setdefault("JAC_EXPERIMENT", "1")  # the library reads experiment knobs only with this set
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_12734_b200 import Jacobi3D

dims = tuple(int(x) for x in os.environ.get("DIMS", "512x512x512").split("x"))
for rep in range(int(os.environ.get("REPS", 2))):
    for bs in os.environ.get("BLOCKS", "16x16x16,8x8x8").split(","):
        blocks = tuple(int(x) for x in bs.split("x"))
        out = []
        for v in os.environ.get("VARS", "3,13").split(","):
            os.environ["JAC_VARIANT"] = v
            with Jacobi3D(dims, blocks) as J:
                J.set_init_hash(1)
                J.step(20)
                J.step(100)
                out.append(f"var {v}: {J.last_step_ms() * 10:.1f} us/iter (variant {J.stats()['sweep_variant']})")
        print(f"blocks {blocks}: " + " | ".join(out), flush=True)
