"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv
--log-file X.csv ...`): launches, total and average time and share per
kernel.  python tools/launch_summary.py X.csv "command" > summary.json"""
import csv
import json
import sys
from collections import defaultdict

rows = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        unit = r["Metric Unit"]
        v = float(r["Metric Value"].replace(",", ""))
        v = v / 1e3 if unit == "ns" else v * 1e3 if unit == "ms" else v  # -> us
        rows.append((r["Kernel Name"], v))
agg = defaultdict(lambda: [0, 0.0])
for k, v in rows:
    agg[k][0] += 1
    agg[k][1] += v
total = sum(v for _, v in rows)
out = {"command": sys.argv[2] if len(sys.argv) > 2 else "", "launches": len(rows), "total_us": round(total, 1),
       "note": "cold-cache, serialised per-launch times (never bench values); shares of the summed kernel time",
       "kernels": [{"kernel": k[:100], "launches": c, "total_us": round(t, 1), "avg_us": round(t / c, 2),
                    "share": round(t / total, 4)}
                   for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])][:40]}
print(json.dumps(out, indent=1))
