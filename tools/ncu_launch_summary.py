"""Summarise an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv` launch list: per kernel name, launches, total
time, total DRAM bytes and DRAM GB/s."""
import csv, collections, sys
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9,
         "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1, "second": 1}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
per, names = collections.defaultdict(dict), {}
for r in rows[1:]:
    per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    names[r[ii]] = r[ki].split("(")[0]
filt = sys.argv[2] if len(sys.argv) > 2 else ""
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    n = names[i]
    if filt not in n:
        continue
    a = agg[n]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tt = sum(v[1] for v in agg.values())
tb = sum(v[2] for v in agg.values())
for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:5d} {t * 1e3:10.3f} ms {b / 1e9:9.2f} GB {b / t / 1e9 if t else 0:8.1f} GB/s  {n}")
print(f"total {tt * 1e3:.3f} ms, {tb / 1e9:.2f} GB DRAM, {tb / tt / 1e9 if tt else 0:.1f} GB/s")
