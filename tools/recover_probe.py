"""How long must the GPU idle after reaching the power cap before a short run is
back in the cold regime?  Drive the sweep into the cap (hash data, ~1.5 s), sleep
X s, then time 60 iterations."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_12734_b200 import Jacobi3D
import bench
dims, blocks, g, label, _ = bench.workload("c2", 1, 8)
J = Jacobi3D(dims, blocks, n_gpus=1, gpu_grid=g)
J.set_init_hash(1)
J.step(100); print("fresh 100:", f"{J.last_step_ms() / 100 * 1e3:.1f}", flush=True)
for x in (0.0, 0.05, 0.1, 0.25, 0.5, 1.0, 2.0, 0.25, 0.5):
    J.step(4000)
    hot = J.last_step_ms() / 4000 * 1e3
    time.sleep(x)
    J.step(60)
    print(f"idle {x:.2f}s: after-cap avg {hot:.1f} -> next 60 iters {J.last_step_ms() / 60 * 1e3:.1f} us/iter", flush=True)
