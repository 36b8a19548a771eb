"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) by kernel (dev tool)."""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = OrderedDict()
for r in rows[1:]:
    us = float(r[iv].replace(",", "")) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[im], 1.0)
    n, t = agg.get(r[ik], (0, 0.0))
    agg[r[ik]] = (n + 1, t + us)
tot = sum(t for _, t in agg.values())
print("| kernel | launches | total us | share |\n|---|---|---|---|")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{k[:80]}` | {n} | {t:.1f} | {t / tot:.3f} |")
