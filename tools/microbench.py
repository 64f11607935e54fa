"""The paper's runtime microbenchmarks on B200:
E1 launch latency, E2 overlap vs ODF, E3 launch rate vs chares x
threads, E4/E5 pipelined NVLink transfers vs ODF with / without an
O(n) consumer kernel.  Prints one JSON object."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_12734_b200 import jacobi3d as J

out = {"device": torch.cuda.get_device_name(0), "n_gpus": torch.cuda.device_count()}
out["E1_launch_latency_us"] = J.jac_mb_launch_latency(0, 5000)
e2 = {}
for total in (32768, 262144, 2097152):
    for odf in (1, 2, 4, 8, 16, 32, 64):
        h, d = J.jac_mb_overlap(total, odf, work=20000)
        e2[f"{total}x{odf}"] = {"threads": total, "odf": odf, "host_us": h, "device_us": d}
out["E2_overlap"] = e2
e3 = {}
for th in (1, 2, 4):
    for ch in (1, 2, 4, 8):
        e3[f"pe{th}_chares{ch}"] = J.jac_mb_launch_rate(ch, th, 0.4)
out["E3_launch_rate_per_s"] = e3
dst = 1 if torch.cuda.device_count() > 1 else 0
e4 = {}
for mb in (0.5, 2, 8, 64):
    nbytes = int(mb * 2 ** 20)
    for odf in (1, 2, 4, 8, 16, 32, 64):
        for comp in (0, 1):
            us = J.jac_mb_pipeline(0, dst, nbytes, odf, comp)
            ub = J.jac_mb_pipeline_batched(0, dst, nbytes, odf, comp)
            vb = J.jac_mb_last_verified_bytes()  # every delivered byte checked
            e4[f"{mb}MiB_odf{odf}_c{comp}"] = {"MiB": mb, "odf": odf, "compute": comp, "us": us,
                                                "GBps": nbytes / us / 1e3, "batched_kernel_us": ub,
                                                "batched_GBps": nbytes / ub / 1e3, "verified_bytes": vb}
out["E4E5_pipeline"] = {"src": 0, "dst": dst, "rows": e4}
print(json.dumps(out))
