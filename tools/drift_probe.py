"""Does per-iteration time depend on the iteration count / field values?  (1 GPU)
Prints per-rep us/iter, average board power over the rep (NVML energy counter), and
SM clock / clock-event reasons sampled during the rep."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import pynvml as N
from paper_2605_12734_b200 import Jacobi3D
import bench

N.nvmlInit(); h = N.nvmlDeviceGetHandleByIndex(0)
print("power limit W:", N.nvmlDeviceGetEnforcedPowerLimit(h) / 1000, flush=True)
dims, blocks, g, label, _ = bench.workload(os.environ.get("CFG", "c2"), 1, int(os.environ.get("ODF", 8)))
J = Jacobi3D(dims, blocks, n_gpus=1, gpu_grid=g, flags=int(os.environ.get("FLAGS", 0)))

def sampled(fn):
    clk, rs, stop = [], [0], threading.Event()
    def loop():
        while not stop.is_set():
            clk.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)); rs[0] |= N.nvmlDeviceGetCurrentClocksEventReasons(h)
            time.sleep(0.002)
    t = threading.Thread(target=loop); t.start()
    e0, t0 = N.nvmlDeviceGetTotalEnergyConsumption(h), time.time()
    fn()
    e1, t1 = N.nvmlDeviceGetTotalEnergyConsumption(h), time.time()
    stop.set(); t.join()
    return (e1 - e0) / 1e3 / (t1 - t0), (min(clk) if clk else 0, int(np.median(clk)) if clk else 0), rs[0]

def reps(tag, k=4, n=100):
    out = []
    for _ in range(k):
        w, c, r = sampled(lambda: J.step(n))
        out.append(f"{J.last_step_ms() / n * 1e3:.1f}[{w:.0f}W {c[0]}/{c[1]}MHz {r:#x}]")
    print(f"{tag:>18}: " + " ".join(out), flush=True)
J.set_init_hash(1); J.step(10)
reps("hash", 6, 200)
nx, ny, nz = dims
box = np.full((nz + 2, ny + 2, nx + 2), 0.5)
J.set_init(box); del box
reps("const 0.5", 3, 200)
J.set_init_hash(1); reps("hash again", 3, 200)
