"""N-GPU coupling A/B (one process, jac_create(n_gpus=N)): C2's 512^3 per GPU at ODF 8,
the fused exchange with the remote items first (default) or spread over the first
f% of the launch order (JAC_REMOTE_SPREAD, experiment knob).  Per setting: ms/iter of
jac_step(K) (device time, max over devices), the per-launch sweep span and the remote
CTAs' peer waits from jac_profile_sweep; settings interleaved, R repetitions."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_12734_b200 as jb

N = int(os.environ.get("N", "4"))
K = int(os.environ.get("K", "50"))
R = int(os.environ.get("R", "3"))
ODF = int(os.environ.get("ODF", "8"))
import bench  # geometry helpers only

dims, blocks, g, _, _ = bench.workload(os.environ.get("CFG", "c2"), N, ODF)
settings = os.environ.get("SPREADS", "first,25,50,80").split(",")
# SETTINGS overrides: ';'-separated env settings 'K=V,K=V' or 'default'
if os.environ.get("SETTINGS"):
    settings = os.environ["SETTINGS"].split(";")
res = {s: [] for s in settings}
for rep in range(R):
    for sp in settings:
        if "=" in sp:
            env = {"JAC_EXPERIMENT": "1", **dict(kv.split("=") for kv in sp.split(","))}
        elif sp in ("first", "default"):
            env = {"JAC_EXPERIMENT": "1", "JAC_REMOTE_SPREAD": "0"} if sp == "first" else {}
        else:
            env = {"JAC_EXPERIMENT": "1", "JAC_REMOTE_SPREAD": sp}
        os.environ.update(env)
        with jb.Jacobi3D(dims, blocks, n_gpus=N, gpu_grid=g) as G:
            for k in env:
                del os.environ[k]
            G.set_init_hash(1)
            G.step(5)
            time.sleep(0.25)
            G.step(K)
            ms = G.last_step_ms() / K
            time.sleep(0.25)
            sw = G.profile_sweep(20)
            st = G.stats()
            res[sp].append((ms, sw, st["peer_wait_ns"], st["peer_wait_max_ns"], st["remote_items"]))
for sp in settings:
    v = res[sp]
    print(f"N={N} ODF={ODF} {sp:28s} ms/iter {statistics.median(x[0] for x in v):.4f} "
          f"sweep {1e3 * statistics.median(x[1] for x in v):.1f} us  peer-wait sum/sweep "
          f"{statistics.median(x[2] for x in v) / 1e3:.1f} us max {max(x[3] for x in v) / 1e3:.1f} us "
          f"remote_items {v[0][4]}", flush=True)
