"""Steady-state (power-capped) sweep time per tile variant on random (hash) data.
For each (ODF, variant): hash init, `settle` iterations to reach the power/clock
equilibrium, then reps of `n` iterations with avg power (NVML energy) and SM clock."""
import os, sys, threading, time
os.environ.setdefault("JAC_EXPERIMENT", "1")  # the library reads experiment knobs only with this set
sys.path.insert(0, os.environ.get("PROBE_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import pynvml as N

N.nvmlInit(); h = N.nvmlDeviceGetHandleByIndex(0)
settle, n, k = int(os.environ.get("SETTLE", 3000)), int(os.environ.get("N", 500)), int(os.environ.get("K", 3))

def sampled(fn):
    clk, rs, stop = [], [0], threading.Event()
    def loop():
        while not stop.is_set():
            clk.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)); rs[0] |= N.nvmlDeviceGetCurrentClocksEventReasons(h)
            time.sleep(0.005)
    t = threading.Thread(target=loop); t.start()
    e0, t0 = N.nvmlDeviceGetTotalEnergyConsumption(h), time.time()
    fn()
    e1, t1 = N.nvmlDeviceGetTotalEnergyConsumption(h), time.time()
    stop.set(); t.join()
    return (e1 - e0) / 1e3 / (t1 - t0), int(np.median(clk)) if clk else 0, rs[0]

def main():
    from paper_2605_12734_b200 import Jacobi3D
    import bench
    cfg = os.environ.get("CFG", "c2")
    for odf in [int(x) for x in os.environ.get("ODFS", "1,8").split(",")]:
        # SETTINGS: ';'-separated list of env settings, each 'K=V,K=V' ('plain' = JAC_F_NO_TMA)
        for var in os.environ.get("SETTINGS", "JAC_VARIANT=0;JAC_VARIANT=5;JAC_VARIANT=12;plain").split(";"):
            flags = 0
            for key in ("JAC_VARIANT", "JAC_ZCHUNK", "JAC_GCOLS", "JAC_ZC", "JAC_L2PROMO", "JAC_PDL", "JAC_YCHUNK"):
                os.environ.pop(key, None)
            if var == "plain":
                flags = 1 << 5
            else:
                for kv in var.split(","):
                    key, val = kv.split("=")
                    os.environ[key] = val
            if cfg == "j2d":
                flags |= 1 << 9
            dims, blocks, g, label, _ = bench.workload(cfg, 1, odf)
            try:
                J = Jacobi3D(dims, blocks, n_gpus=1, gpu_grid=g, flags=flags)
            except Exception as e:
                print(f"odf {odf} var {var}: {e}", flush=True); continue
            J.set_init_hash(1)
            J.step(10)
            cold = []
            for _ in range(3):  # pre-throttle regime: constant -> hash switch resets the clocks
                J.set_init_hash(1); J.step(5); J.step(60); cold.append(J.last_step_ms() / 60 * 1e3)
            J.step(settle)
            out = []
            for _ in range(k):
                w, c, r = sampled(lambda: J.step(n))
                out.append(f"{J.last_step_ms() / n * 1e3:.1f}us[{w:.0f}W {c}MHz {r:#x}]")
            print(f"{label} {var:>28}: cold {min(cold):.1f}us | steady " + " ".join(out), flush=True)
            J.close()
main()
