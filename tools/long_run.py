"""Minute-long run of the bench decomposition (512^3 ODF 8, random data): GLUP/s,
SM clock and GPU temperature per window of WIN iterations."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml as N
from paper_2605_12734_b200 import Jacobi3D

N.nvmlInit(); h = N.nvmlDeviceGetHandleByIndex(0)
win, wins = int(os.environ.get("WIN", 10000)), int(os.environ.get("WINS", 17))
with Jacobi3D((512, 512, 512), (2, 2, 2)) as J:
    J.set_init_hash(1)
    J.step(10)
    for w in range(wins):
        clk, tmp, stop = [], [], threading.Event()
        def loop():
            while not stop.is_set():
                clk.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)); tmp.append(N.nvmlDeviceGetTemperature(h, 0))
                time.sleep(0.02)
        th = threading.Thread(target=loop); th.start()
        J.step(win)
        stop.set(); th.join()
        us = J.last_step_ms() / win * 1e3
        print(f"window {w:2d}: {us:6.1f} us/iter  {512**3 / us / 1e3:6.1f} GLUP/s  sm {sorted(clk)[len(clk) // 2]} MHz  "
              f"temp {max(tmp)} C", flush=True)
