"""Per-source-line instruction and stall shares of one kernel from an ncu
--set full capture: joins the SASS page (ncu -i X --page source --csv
--print-source sass) with nvdisasm -g line info of the same cubin
(cuobjdump -xelf all libsait_b200.so; nvdisasm -g -c spgemm.sm_100a.cubin).
python tools/ncu_lines.py <nvdisasm.sass> <mangled-name regex> <sass.csv> <source.cu> [top]"""
import csv, re, sys, collections
sass_file, func_pat, ncu_csv, src = sys.argv[1:5]
lines = open(sass_file).read().splitlines()
start = None
for i, l in enumerate(lines):
    if l.startswith("//---------------------") and re.search(func_pat, l):
        start = i; break
off2line = {}; cur = None
for l in lines[start+1:]:
    if l.startswith("//---------------------"): break
    m = re.search(r'//## File ".*", line (\d+)', l)
    if m: cur = int(m.group(1)); continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
    if m: off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(ncu_csv)))
hdr = rows[1]; data = [r for r in rows[2:] if len(r) > 5 and r[0].startswith("0x")]
iE = hdr.index("Instructions Executed"); iW = hdr.index("Warp Stall Sampling (All Samples)")
base = int(data[0][0], 16)
agg_e = collections.Counter(); agg_w = collections.Counter()
for r in data:
    off = int(r[0], 16) - base
    ln = off2line.get(off)
    agg_e[ln] += int(float(r[iE] or 0)); agg_w[ln] += int(float(r[iW] or 0))
te = sum(agg_e.values()); tw = sum(agg_w.values())
srcl = open(src).read().splitlines()
print(f"total inst {te} samples {tw}; mapped offsets {len(off2line)} of {len(data)}")
for ln, w in agg_w.most_common(int(sys.argv[5]) if len(sys.argv) > 5 else 30):
    t = srcl[ln-1].strip()[:80] if ln else "?"
    print(f"{ln}: inst {agg_e[ln]/te*100:5.1f}%  stall {w/tw*100:5.1f}%  | {t}")
