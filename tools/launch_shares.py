"""Per-kernel shares from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import json
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("void epd::", "").strip()
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) / 1e3  # ns -> us
total = sum(v[1] for v in agg.values())
out = {"source": sys.argv[2] if len(sys.argv) > 2 else "", "total_us": total, "kernels": {}}
for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out["kernels"][k] = {"launches": c, "us_per_launch": us / c, "share": us / total}
print(json.dumps(out, indent=1))
