"""(JAC_EXPERIMENT=1 JAC_STAGE_PITCHED=1: the pitched staging path.)  Breakdown of the e2e job (bench.py run_e2e): jac_set_init_box, jac_step(K),
jac_get_field_box with pinned host buffers, each timed on the host, next to plain
linear pinned H2D / D2H copies of the same byte counts (torch)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import jac_inputs as JI
from paper_2605_12734_b200 import Jacobi3D

N = int(os.environ.get("N", "512"))
B = tuple(int(x) for x in os.environ.get("BLOCKS", "2x2x2").split("x"))
K = int(os.environ.get("K", "20"))
dims = (N, N, N)
origin, extent = (0, 0, 0), (N + 2, N + 2, N + 2)
host_in = torch.empty((N + 2,) * 3, dtype=torch.float64, pin_memory=True)
host_in.numpy()[...] = JI.hash_box(*dims, origin, extent, seed=1)
INTERIOR = os.environ.get("INTERIOR") == "1"  # read back a box of just the interiors
host_out = torch.empty_like(host_in, pin_memory=True)
out_box = host_out[1:-1, 1:-1, 1:-1].contiguous().pin_memory() if INTERIOR else host_out
out_origin = (1, 1, 1) if INTERIOR else origin
dev = torch.empty_like(host_in, device="cuda")
for r in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); dev.copy_(host_in, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter(); host_out.copy_(dev, non_blocking=True); torch.cuda.synchronize()
    t2 = time.perf_counter()
    gb = host_in.numel() * 8 / 1e9
    print(f"torch linear: H2D {(t1-t0)*1e3:.2f} ms ({gb/(t1-t0):.1f} GB/s)  D2H {(t2-t1)*1e3:.2f} ms ({gb/(t2-t1):.1f} GB/s)", flush=True)
del dev
with Jacobi3D(dims, B) as J:
    J.set_init_box(host_in.numpy(), origin)
    J.step(K)
    for r in range(3):
        t0 = time.perf_counter(); J.set_init_box(host_in.numpy(), origin)
        t1 = time.perf_counter(); J.step(K)
        t2 = time.perf_counter(); J.field_box(out_box.numpy(), out_origin)
        t3 = time.perf_counter()
        print(f"jac: set_init_box {(t1-t0)*1e3:.2f} ms  step({K}) {(t2-t1)*1e3:.2f} ms  field_box {(t3-t2)*1e3:.2f} ms"
              f"  total {(t3-t0)*1e3:.2f} ms -> {N**3*K/(t3-t0)/1e9:.1f} GLUP/s", flush=True)
