"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
iN, iM, iU, iV, iID = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
per = defaultdict(dict)
names = {}
for r in rows[start + 1:]:
    if len(r) <= iV:
        continue
    v = float(r[iV].replace(",", ""))
    u = r[iU]
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3,
             "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
    per[r[iID]][r[iM]] = v * scale
    names[r[iID]] = r[iN].split("(")[0]
agg = defaultdict(lambda: [0, 0.0, 0.0])
for k, m in per.items():
    a = agg[names[k]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0)
    a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':58s} {'n':>4s} {'mean us':>9s} {'share':>6s} {'GB/s':>8s} {'MB/launch':>10s}")
for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n[:58]:58s} {c:4d} {t / c:9.2f} {t / tot:6.1%} {b / (t * 1e-6) / 1e9 if t else 0:8.0f} {b / c / 1e6:10.2f}")
