"""Same-process repeat of the ODF sweep (allocation / thermal drift check)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml as N
import paper_2605_12734_b200 as jb
N.nvmlInit(); h = N.nvmlDeviceGetHandleByIndex(0)
keep = os.environ.get("KEEP") == "1"
held = []
for rep in range(3):
    for blocks in [(2, 2, 2), (1, 1, 1), (2, 2, 4), (4, 4, 4), (2, 2, 2)]:
        s = jb.Jacobi3D((512, 512, 512), blocks)
        s.set_init_hash(1); s.step(6); s.step(50)
        ms = s.last_step_ms() / 50
        t = N.nvmlDeviceGetTemperature(h, 0)
        try:
            mt = N.nvmlDeviceGetFieldValues(h, [N.NVML_FI_DEV_MEMORY_TEMP])[0].value.uiVal
        except Exception:
            mt = -1
        mclk = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_MEM)
        print(f"rep {rep} blocks {blocks}: {ms*1e3:7.1f} us  gpuT={t} memT={mt} memclk={mclk}", flush=True)
        if keep:
            held.append(s)
        else:
            s.close()
