"""3-D z-chunk length (JAC_ZCHUNK) and tile variant per block shape at 512^3: graph-
replayed us/iter, settings interleaved, median of R.  SETS='16;8;32;64' (';'-separated
settings, each 'K=V,K=V' or 'default')."""
import os, statistics, sys, time
os.environ.setdefault("JAC_EXPERIMENT", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_12734_b200 import Jacobi3D

dims = tuple(int(x) for x in os.environ.get("DIMS", "512x512x512").split("x"))
R = int(os.environ.get("R", "3"))
for bs in os.environ.get("BLOCKS", "1x1x1,2x2x2,4x4x4,8x8x8").split(","):
    blocks = tuple(int(x) for x in bs.split("x"))
    sets = os.environ.get("SETS", "default;JAC_ZCHUNK=8;JAC_ZCHUNK=12;JAC_ZCHUNK=24;JAC_ZCHUNK=32").split(";")
    res = {k: [] for k in sets}
    for _ in range(R):
        for st in sets:
            for k in ("JAC_ZCHUNK", "JAC_VARIANT", "JAC_GCOLS"):
                os.environ.pop(k, None)
            if st != "default":
                for kv in st.split(","):
                    k, v = kv.split("=")
                    os.environ[k] = v
            with Jacobi3D(dims, blocks) as J:
                J.set_init_hash(1)
                J.step(10)
                time.sleep(0.2)
                J.step(100)
                res[st].append(J.last_step_ms() * 10)
    base = statistics.median(res[sets[0]])
    print(f"blocks {blocks}: " + "  ".join(f"{k}: {statistics.median(v):.1f} us ({statistics.median(v) / base - 1:+.1%})"
                                           for k, v in res.items()), flush=True)
