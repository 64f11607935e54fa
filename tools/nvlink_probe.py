"""One process, N GPUs (jac_create(n_gpus=N)), C2's 512^3 per GPU at ODF 8, launched
WITHOUT graphs so the sweeps of the devices are enqueued interleaved (d0 it0, d1 it0,
d0 it1, ...): under ncu (which serialises launches) every sweep's peers have already
signalled.  For ncu's NVLink counters of the fused sweep+exchange kernel:
  ncu --metrics nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,gpu__time_duration.sum \\
      -k regex:sweep_tma -s 4 -c 4 python tools/nvlink_probe.py
Prints the library's remote bytes per GPU and iteration for comparison."""
import os
import sys

sys.path.insert(0, os.environ.get("PROBE_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("JAC_EXPERIMENT", "1")
os.environ.setdefault("JAC_AUTOTUNE", "0")  # no create-time timing sweeps in the launch list
import paper_2605_12734_b200 as jb
from paper_2605_12734_b200 import jacobi3d as J

N = int(os.environ.get("N", "2"))
box = int(os.environ.get("BOX", "512"))
g = {2: (1, 1, 2), 4: (1, 2, 2), 8: (2, 2, 2)}[N]
if os.environ.get("GRID"):  # e.g. GRID=2x1x1: an x split (remote x faces: the x-ghost arrays)
    g = tuple(int(v) for v in os.environ["GRID"].split("x"))
dims = tuple(box * g[d] for d in range(3))
blocks = tuple(2 * g[d] for d in range(3))
with jb.Jacobi3D(dims, blocks, n_gpus=N, gpu_grid=g, flags=J.JAC_F_NO_GRAPH) as G:
    G.set_init_hash(1)
    G.step(int(os.environ.get("K", "6")))
    st = G.stats()
    print(f"N={N} dims={dims} blocks={blocks} remote_bytes_per_gpu_per_iter={st['remote_bytes'] / N:.0f} "
          f"remote_faces_per_gpu={st['remote_faces'] / N:.0f} kernels_per_iter={st['kernels_per_iter']}", flush=True)
