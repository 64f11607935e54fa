"""Graph-replayed iteration time with and without programmatic dependent launch,
for small (launch-bound) and large grids.  JAC_PDL is read at jac_create."""
import os, sys
os.environ.setdefault("JAC_EXPERIMENT", "1")  # the library reads experiment knobs only with this set
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_12734_b200 import Jacobi3D

CASES = [((64, 64, 64), (2, 2, 2), 0, 2000), ((128, 128, 128), (2, 2, 2), 0, 1000),
         ((512, 512, 512), (1, 1, 1), 0, 200), ((512, 512, 512), (2, 2, 2), 0, 200),
         ((512, 512, 512), (16, 16, 16), 0, 100), ((32768, 32768, 1), (2, 4, 1), 1 << 9, 40)]
for rep in range(2):
    for dims, blocks, flags, n in CASES:
        out = []
        for pdl in ("1", "0"):
            os.environ["JAC_PDL"] = pdl
            with Jacobi3D(dims, blocks, flags=flags) as J:
                J.set_init_hash(1)
                J.step(20)
                J.step(n)
                out.append(J.last_step_ms() / n * 1e3)
        print(f"{dims} {blocks}: pdl {out[0]:.2f} us/iter  no-pdl {out[1]:.2f} us/iter  ({out[1] / out[0] - 1:+.1%})",
              flush=True)
