"""Jacobi2D x-band width (x tiles per band of the work list, JAC_XBAND; 0 = whole
block width) vs block width: graph-replayed us/iter, settings interleaved, median of R."""
import os, statistics, sys, time
os.environ.setdefault("JAC_EXPERIMENT", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_12734_b200 import Jacobi2D

cases = []
for c in os.environ.get("DIMS", "131072x16384,131072x32768,65536x32768,32768x32768").split(","):
    d, _, b = c.partition(":")
    cases.append((tuple(map(int, d.split("x"))), tuple(map(int, b.split("x"))) if b else (1, 1)))
chunks = os.environ.get("BANDS", "0,256,512,1024").split(",")
R = int(os.environ.get("R", "3"))
for dims, blocks in cases:
    res = {c: [] for c in chunks}
    for _ in range(R):
        for ch in chunks:
            os.environ["JAC_XBAND"] = ch
            with Jacobi2D(dims, blocks) as J:
                J.set_init_hash(1)
                J.step(10)
                time.sleep(0.2)
                n = max(10, int(4e9 / (dims[0] * dims[1])))
                J.step(n)
                res[ch].append(J.last_step_ms() / n * 1e3)
    print(f"{dims[0]}x{dims[1]} blocks {blocks}: " + "  ".join(f"xband {c}: {statistics.median(v):.1f} us" for c, v in res.items()), flush=True)
