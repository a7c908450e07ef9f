"""Print the hottest SASS lines (warp-stall samples) of an ncu report's
source page: python tools/ncu_hot.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
# first line is the kernel name row; the header follows
blocks = []
cur = None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = [ln]
        blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
for b in blocks[:1]:
    print(b[0][:150])
    rows = list(csv.reader(io.StringIO("\n".join(b[1:]))))
    hdr = rows[0]
    i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    extra = [h for h in hdr if h.startswith("stall_") or "Stall" in h]
    data = rows[1:]
    tot = sum(float(r[i_s] or 0) for r in data)
    data.sort(key=lambda r: -float(r[i_s] or 0))
    for r in data[:top]:
        print(f"{float(r[i_s]) / tot * 100:5.1f}%  {r[0][-5:]}  {r[i_src].strip()[:80]}")
    print("columns:", [h for h in hdr][:60])
