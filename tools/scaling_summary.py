"""Assemble bench.py JSON lines (files named bench_<cfg>_n<N>.json) into one scaling
summary: per (config, N) the bench value plus speed-up and efficiency against N=1
(weak: value_N / (N * value_1); strong: (value_N / value_1) / N).
python tools/scaling_summary.py OUT.json FILE..."""
import json
import os
import re
import sys


def main():
    out, files = sys.argv[1], sys.argv[2:]
    lines = {}
    for f in files:
        m = re.match(r"bench_(.+)_n(\d+)\.json$", os.path.basename(f))
        if not m:
            continue
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
        except (ValueError, IndexError):
            continue
        if "value" not in d or d.get("impl") == "reference":
            continue
        lines[(m.group(1), int(m.group(2)))] = d
    res = {}
    for (cfg, n), d in sorted(lines.items()):
        base = lines.get((cfg, 1))
        e = {k: d.get(k) for k in ("value", "unit", "ms_per_step", "n_gpus", "scaling", "config", "gpu_launches",
                                   "clocks", "exchange")}
        e["roofline_frac"] = (d.get("roofline") or {}).get("frac")
        for key in ("exchange_ablations", "ablation_nccl_sendrecv"):
            if d.get(key):
                e[key] = d[key]
        if base:
            sp = d["value"] / base["value"]
            e["speedup_vs_1gpu"] = sp
            e["efficiency"] = sp / n if d.get("scaling") == "strong" else d["value"] / (n * base["value"])
        res[f"{cfg}_n{n}"] = e
    json.dump(res, open(out, "w"), indent=1)
    for k, e in res.items():
        print(f"{k:14s} {e['value']:9.1f} {e['unit']}  {1e3 * e['ms_per_step']:8.1f} us/step  "
              f"eff {e.get('efficiency', float('nan')):.3f}")


if __name__ == "__main__":
    main()
