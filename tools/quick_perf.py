"""Quick ODF sweep timing at 512^3 (development helper; bench.py is the contract)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_12734_b200 as jb
from bench import ClockSampler

n = int(os.environ.get("N", 512))
iters = int(os.environ.get("ITERS", 50))
flags = int(os.environ.get("FLAGS", 0))
odfs = [(1,1,1),(1,1,2),(1,2,2),(2,2,2),(2,2,4),(2,4,4),(4,4,4)]
only = os.environ.get("ODFS")
if only:
    odfs = [o for o in odfs if str(o[0]*o[1]*o[2]) in only.split(",")]
for blocks in odfs:
    with jb.Jacobi3D((n, n, n), blocks, flags=flags) as s:
        s.set_init_hash(1)
        s.step(6)
        cs = ClockSampler(0)
        with cs:
            s.step(iters)
        ms = s.last_step_ms() / iters
        sw = s.profile_sweep(10)
        glups = n**3 / (ms * 1e6)
        c = cs.summary()
        print(f"ODF {blocks[0]*blocks[1]*blocks[2]:3d} {blocks}: {ms*1e3:8.1f} us/iter {glups:7.1f} GLUP/s "
              f"{16*glups:6.0f} GB/s sweep {sw*1e3:7.1f} us sm={c['sm_mhz']} {c['reasons']}", flush=True)
