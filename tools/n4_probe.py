"""Where does the N=4 weak-scaling loss come from?  On N GPUs of one box, C2's 512^3
per GPU at ODF 8 (1x2x2 grid at N=4):
  indep     N independent 1-GPU contexts (no exchange, no coupling) running at once
  solo      one 1-GPU context alone on GPU 0
  fused     jac_create(n_gpus=N), default (in-sweep peer stores + flag handshake)
  nofused   same, cross-GPU ordering by the barrier kernel (JAC_NO_FUSED_SYNC)
  skip      same, exchange skipped (barrier kernel only; WRONG results)
Prints ms/iter (device time of jac_step(K), max over devices) and the per-launch
sweep span of jac_profile_sweep, median of R repetitions."""
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_12734_b200 as jb
from paper_2605_12734_b200 import jacobi3d as J

N = int(os.environ.get("N", "4"))
K = int(os.environ.get("K", "50"))
R = int(os.environ.get("R", "5"))
box = 512
gz, gy = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (2, 2)}[N]
gx = 2 if N == 8 else 1


def one_gpu_ctx(dev):
    c = jb.Jacobi3D((box, box, box), (2, 2, 2), n_gpus=1, rank=0, device=dev)
    J.jac_import_ipc(c.ctx, [J.jac_export_ipc(c.ctx)])
    c.set_init_hash(1)
    return c


def timed(ctxs):
    """steps K on every context concurrently (one thread each); max device ms/iter."""
    res = [0.0] * len(ctxs)

    def run(i):
        ctxs[i].step(K)
        res[i] = ctxs[i].last_step_ms() / K
    for c in ctxs:
        c.step(5)
    time.sleep(0.25)
    th = [threading.Thread(target=run, args=(i,)) for i in range(len(ctxs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return max(res)


def report(name, vals, spans=None):
    s = f"{name:8s} ms/iter median {statistics.median(vals):.4f} min {min(vals):.4f} max {max(vals):.4f}"
    if spans:
        s += f"  sweep span median {statistics.median(spans) * 1e3:.1f} us"
    print(s, flush=True)


ctxs = [one_gpu_ctx(d) for d in range(N)]
report("indep", [timed(ctxs) for _ in range(R)])
report("solo", [timed(ctxs[:1]) for _ in range(R)])
for c in ctxs:
    c.close()
dims = (box * gx, box * gy, box * gz)
blocks = (2 * gx, 2 * gy, 2 * gz)
for name, flags, env in [("fused", 0, {}), ("nofused", 0, {"JAC_EXPERIMENT": "1", "JAC_NO_FUSED_SYNC": "1"}),
                         ("skip", J.JAC_F_SKIP_EXCHANGE, {})]:
    os.environ.update(env)
    with jb.Jacobi3D(dims, blocks, n_gpus=N, flags=flags) as G:
        for k in env:
            del os.environ[k]
        G.set_init_hash(1)
        vals, spans = [], []
        for _ in range(R):
            G.step(5)
            time.sleep(0.25)
            G.step(K)
            vals.append(G.last_step_ms() / K)
            time.sleep(0.25)
            spans.append(G.profile_sweep(20))
        report(name, vals, spans)
