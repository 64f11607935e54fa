"""Multi-rank timing of one decomposition (torchrun).  FLAGS env = jac flags."""
import os, sys
os.environ.setdefault("JAC_EXPERIMENT", "1")  # the library reads experiment knobs only with this set
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2605_12734_b200.dist import create_rank_context, destroy_rank_context
import bench

local = int(os.environ.get("LOCAL_RANK", 0)); torch.cuda.set_device(local)
dist.init_process_group("nccl")
n = dist.get_world_size()
flags = int(os.environ.get("FLAGS", 0))
cfg = os.environ.get("CFG", "c2")
dims, blocks, g, label, _ = bench.workload(cfg, n, int(os.environ.get("ODF", 8)))
J = create_rank_context(dims, blocks, gpu_grid=g, flags=flags, device=local)
J.set_init_hash(1)
J.step(10)
res = []
cs = bench.ClockSampler(local)
for rep in range(int(os.environ.get("REPS", 3))):
    dist.barrier(); torch.cuda.synchronize()
    with cs:
        J.step(100)
    t = torch.tensor([J.last_step_ms() / 100], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    res.append(t.item() * 1e3)
sw = J.profile_sweep(30)
t = torch.tensor([sw * 1e3], device="cuda"); dist.all_reduce(t, op=dist.ReduceOp.MAX)
if dist.get_rank() == 0:
    print(f"N={n} {label} flags={flags} nofused={os.environ.get('JAC_NO_FUSED_SYNC','')} us/iter={['%.1f' % r for r in res]} sweep_median={t.item():.1f} clocks={cs.summary()}", flush=True)
destroy_rank_context(J)
dist.destroy_process_group()
