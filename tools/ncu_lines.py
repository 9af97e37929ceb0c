"""Dev helper: attribute ncu warp-stall samples of one kernel to CUDA source
lines. Inputs: the SASS source page (ncu -i rep --page source --csv) and
nvdisasm -g -c output of the cubin that holds the kernel.
  python tools/ncu_lines.py sass.csv nvdisasm.txt '<mangled kernel name>' [top]"""
import csv
import re
import sys
from collections import defaultdict

sass_csv, dis, fn = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 60
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
data = rows[2:]
col = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
# instruction -> line from nvdisasm
lines = []
cur = None
infn = False
for ln in open(dis):
    if ln.startswith(".text."):
        infn = ln.strip() == ".text." + fn + ":"
        continue
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
        lines.append(cur)
print("instructions: ncu", len(data), "nvdisasm", len(lines))
agg = defaultdict(lambda: defaultdict(int))
tot = defaultdict(int)
for r, l in zip(data, lines):
    for h in reasons:
        v = int(r[col[h]] or 0)
        if v:
            agg[l][h] += v
            tot[h] += v
print("totals:", {h: v for h, v in sorted(tot.items(), key=lambda x: -x[1])})
work = [h for h in reasons if h not in ("stall_barrier",)]
rank = sorted(agg.items(), key=lambda kv: -sum(kv[1][h] for h in work))
allw = sum(sum(v[h] for h in work) for v in agg.values())
print("non-barrier samples:", allw)
for l, v in rank[:top]:
    w = sum(v[h] for h in work)
    det = ", ".join(f"{h[6:]}={c}" for h, c in sorted(v.items(), key=lambda x: -x[1])[:4])
    print(f"{l[0]}:{l[1]:5d}  {w:6d} ({100.0 * w / allw:4.1f}%)  {det}")

# ---- bucketed by source region (event_kernel.cu line ranges)
if len(sys.argv) > 5:
    step = int(sys.argv[5])
    b = defaultdict(lambda: defaultdict(int))
    for l, v in agg.items():
        key = (l[0], (l[1] // step) * step) if l and l[0] == "event_kernel.cu" else (l[0] if l else "?", 0)
        for h, c in v.items():
            b[key][h] += c
    print("\nby region:")
    for key, v in sorted(b.items(), key=lambda kv: (kv[0][0] != "event_kernel.cu", kv[0][1])):
        w = sum(v[h] for h in work)
        if w < 20:
            continue
        det = ", ".join(f"{h[6:]}={c}" for h, c in sorted(v.items(), key=lambda x: -x[1])[:5])
        print(f"{key[0]}:{key[1]:5d}+  {w:6d} ({100.0 * w / allw:4.1f}%)  {det}")
