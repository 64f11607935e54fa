"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import csv, io, json, sys
from collections import defaultdict

text = open(sys.argv[1]).read()
text = text[text.index('"ID"'):]
rows = list(csv.reader(io.StringIO(text)))
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3}
agg = defaultdict(list)
for r in rows[1:]:
    agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")) * scale[r[ui]])
out = {}
tot = sum(sum(v) for v in agg.values())
for k, v in agg.items():
    out[k] = {"launches": len(v), "mean_us": sum(v) / len(v), "total_us": sum(v), "share": sum(v) / tot}
print(json.dumps(out, indent=1))
