"""Sustained HBM copy bandwidth vs data content on 1 GPU: each pattern is copied for
~SECS seconds; per ~100 ms window prints GB/s, SM clock and clock-event reasons.
Answers whether a plain copy of random data is itself power capped (the sustained
ceiling the sweep should be compared with)."""
import os, time, threading, torch, pynvml as N
N.nvmlInit(); h = N.nvmlDeviceGetHandleByIndex(0)
n = 1 << 28  # 2 GiB of fp64 per buffer
secs = float(os.environ.get("SECS", 3))
src = torch.empty(n, dtype=torch.float64, device="cuda"); dst = torch.empty_like(src)
def run(tag):
    out, per = [], 150
    t_end = time.time() + secs
    while time.time() < t_end:
        clk, rs, stop = [], [0], threading.Event()
        def loop():
            while not stop.is_set():
                clk.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)); rs[0] |= N.nvmlDeviceGetCurrentClocksEventReasons(h)
                time.sleep(0.005)
        th = threading.Thread(target=loop); th.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(per):
            dst.copy_(src)
        e1.record(); e1.synchronize(); stop.set(); th.join()
        out.append(f"{2 * n * 8 * per / (e0.elapsed_time(e1) * 1e-3) / 1e9:.0f}/{min(clk) if clk else 0}{'c' if rs[0] & 4 else ''}")
    print(f"{tag:>8} (GB/s / min SM MHz, c = sw power cap): " + " ".join(out), flush=True)
for tag, fill in [("zeros", lambda: src.zero_()), ("random", lambda: src.uniform_()), ("zeros", lambda: src.zero_()),
                  ("random", lambda: src.uniform_())]:
    fill(); torch.cuda.synchronize(); run(tag)
