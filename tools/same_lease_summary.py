"""Summarise a same-lease campaign (tools/run_campaign4b.sh, PFX=<p>): gpurun_out/<p>_*.json
-> one JSON with every line and the derived weak-scaling efficiencies / strong speed-ups.
python tools/same_lease_summary.py PFX OUT.json "description" """
import glob
import json
import os
import sys

pfx, out_path, desc = sys.argv[1], sys.argv[2], sys.argv[3]
out = {"box": desc, "command": f"PFX={pfx} tools/run_campaign4b.sh", "lines": {}}
for f in sorted(glob.glob(f"gpurun_out/{pfx}_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except (ValueError, IndexError):
        continue
    if "value" not in d:
        continue
    s = d.get("sustained_power_capped") or {}
    out["lines"][os.path.basename(f)[:-5]] = {
        "workload": d["config"]["workload"], "n_gpus": d["n_gpus"], "gpu_grid": d["config"].get("gpu_grid"),
        "blocks": d["config"].get("blocks"), "glups": d["value"], "ms_per_iter": d["ms_per_step"],
        "roofline_frac": d["roofline"]["frac"], "sustained_glups": s.get("value"), "launch": d.get("launch"),
        "rank_ms_per_step": d.get("rank_ms_per_step"), "exchange_ablations": d.get("exchange_ablations"),
        "clocks": d.get("clocks"), "e2e": d.get("e2e")}
L = out["lines"]


def eff(a, b, n, strong=False):
    if a not in L or b not in L:
        return None
    r = L[b]["glups"] / (n * L[a]["glups"])
    return r * n if strong else r


p = pfx
out["derived"] = {
    "c2_weak_eff_one_process": {"n2": eff(f"{p}_c2_n1", f"{p}_c2_n2", 2), "n4": eff(f"{p}_c2_n1", f"{p}_c2_n4", 4)},
    "c2_weak_eff_torchrun": {"n2": eff(f"{p}_c2_n1", f"{p}_c2tr_n2", 2), "n4": eff(f"{p}_c2_n1", f"{p}_c2tr_n4", 4)},
    "c3_weak_eff": {"n2": eff(f"{p}_c3_n1", f"{p}_c3_n2", 2), "n4": eff(f"{p}_c3_n1", f"{p}_c3_n4", 4)},
    "j2d_weak_eff": {"n2": eff(f"{p}_j2d_n1", f"{p}_j2d_n2", 2), "n4": eff(f"{p}_j2d_n1", f"{p}_j2d_n4", 4)},
    "c5_strong_speedup": {"n2": eff(f"{p}_c5_n1", f"{p}_c5_n2", 2, True), "n4": eff(f"{p}_c5_n1", f"{p}_c5_n4", 4, True)},
    "c4_odf16_strong_speedup": {"n2": eff(f"{p}_c4_n1", f"{p}_c4_n2", 2, True), "n4": eff(f"{p}_c4_n1", f"{p}_c4_n4", 4, True)},
}
if f"{p}_j2ds_odf1_n2" in L and f"{p}_j2ds_odf1_n4" in L:
    out["derived"]["j2d_strong_2_to_4"] = {
        o: L[f"{p}_j2ds_odf{o}_n4"]["glups"] / L[f"{p}_j2ds_odf{o}_n2"]["glups"] for o in (1, 16)
        if f"{p}_j2ds_odf{o}_n4" in L and f"{p}_j2ds_odf{o}_n2" in L}
json.dump(out, open(out_path, "w"), indent=1)
print(json.dumps(out["derived"], indent=1))
