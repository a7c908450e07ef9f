"""Summarise an ncu --csv metrics log of tools/ncu_apply.py: per kernel, the
mean DRAM bytes (read + write) and duration per launch, skipping the first
`--skip` launches of each kernel (warm-up).  Usage:
  python tools/ncu_traffic.py log.csv [--skip 2] [--stream-bytes B_L B_U] > summary.json"""
import argparse
import csv
import io
import json
import re

ap = argparse.ArgumentParser()
ap.add_argument("log")
ap.add_argument("--skip", type=int, default=2)
ap.add_argument("--stream-bytes", type=int, nargs=2, default=None)
a = ap.parse_args()
txt = open(a.log).read()
start = txt.find('"ID"')
rows = list(csv.DictReader(io.StringIO(txt[start:])))
by = {}
for r in rows:
    key = (r["ID"], r["Kernel Name"])
    by.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
launches = []
for (lid, name), m in sorted(by.items(), key=lambda kv: int(kv[0][0])):
    launches.append({"id": int(lid), "kernel": re.sub(r"\(.*", "", name)[:80],
                     "dram_bytes": m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0),
                     "dram_read": m.get("dram__bytes_read.sum"), "dram_write": m.get("dram__bytes_write.sum"),
                     "ns": m.get("gpu__time_duration.sum"), "l2_hit_pct": m.get("lts__t_sector_hit_rate.pct")})
use = launches[2 * a.skip:]
mean = lambda k: sum(x[k] for x in use) / max(1, len(use))  # noqa: E731
out = {"source": a.log, "launches_used": len(use), "skipped": 2 * a.skip,
       "dram_bytes_per_launch_mean": mean("dram_bytes"), "ns_per_launch_mean": mean("ns"),
       "dram_gbs_during_launch": mean("dram_bytes") / mean("ns"),
       "l2_hit_pct_mean": mean("l2_hit_pct") if all(x["l2_hit_pct"] is not None for x in use) else None,
       "launches": launches}
if a.stream_bytes:
    out["format_stream_bytes_per_launch_mean"] = sum(a.stream_bytes) / 2
    out["dram_over_format_bytes"] = out["dram_bytes_per_launch_mean"] / out["format_stream_bytes_per_launch_mean"]
print(json.dumps(out, indent=1))
