"""Jacobi2D row pitch (JAC_PALIGN: row pitch rounded up to a multiple of this many
doubles) on wide blocks: graph-replayed us/iter, interleaved, median of R."""
import os, statistics, sys, time
os.environ.setdefault("JAC_EXPERIMENT", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_12734_b200 import Jacobi2D

R = int(os.environ.get("R", "3"))
for case in os.environ.get("DIMS", "131072x16384,32768x32768").split(","):
    dims = tuple(int(v) for v in case.split("x"))
    sets = os.environ.get("ALIGNS", "4,36,132,1028").split(",")
    res = {a: [] for a in sets}
    for _ in range(R):
        for al in sets:
            os.environ["JAC_PALIGN"] = al
            with Jacobi2D(dims, (1, 1)) as J:
                J.set_init_hash(1)
                J.step(10)
                time.sleep(0.2)
                n = max(10, int(4e9 / (dims[0] * dims[1])))
                J.step(n)
                res[al].append(J.last_step_ms() / n * 1e3)
    print(f"{case}: " + "  ".join(f"palign {a}: {statistics.median(v):.1f} us" for a, v in res.items()), flush=True)
