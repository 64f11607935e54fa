"""NEXT-2 A/B: batched table + graph vs paper-style per-block streams at ODF 1..4096
(512^3 on one GPU).  python tools/paper_style.py [iters]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_12734_b200 as jb
from paper_2605_12734_b200 import jacobi3d as J

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rows = []
for blocks in [(1, 1, 1), (2, 2, 2), (2, 2, 4), (4, 4, 4), (8, 8, 8), (16, 16, 16)]:
    odf = blocks[0] * blocks[1] * blocks[2]
    for mode, flags, threads in [("batched", 0, 1), ("per_block", J.JAC_F_PER_BLOCK, 1), ("per_block", J.JAC_F_PER_BLOCK, 4)]:
        n = iters if (mode == "batched" or odf <= 512) else max(2, iters // 10)
        with jb.Jacobi3D((512, 512, 512), blocks, flags=flags) as s:
            s.set_option(J.JAC_OPT_LAUNCH_THREADS, threads)
            s.set_init_hash(1)
            s.step(2)
            t0 = time.perf_counter()
            s.step(n)
            wall = time.perf_counter() - t0
            ms = s.last_step_ms() / n
            st = s.stats()
        r = {"odf": odf, "mode": mode, "launch_threads": threads, "iters": n, "ms_per_iter": ms,
             "wall_ms_per_iter": 1e3 * wall / n, "glups": 512 ** 3 / (ms * 1e6), "kernels_per_iter": st["kernels_per_iter"]}
        rows.append(r)
        print(json.dumps(r), flush=True)
