"""Dev tool: stall-reason totals and top SASS instructions of the first kernel in an ncu
source-page CSV (ncu -i REP --page source --csv --print-source sass > file). Usage:
ncu_sass_top.py CSV [N] [lo_hex hi_hex]  (optional address window, offsets from the kernel start)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr):
        data.append(r)
ci = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][0], 16)
tot = lambda r: sum(int(r[ci[k]] or 0) for k in reasons)  # noqa: E731
T = sum(tot(r) for r in data) or 1
tr = collections.Counter()
for r in data:
    for k in reasons:
        tr[k] += int(r[ci[k]] or 0)
print("totals", ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in tr.most_common(10)))
sel = data
if len(sys.argv) > 4:
    lo, hi = int(sys.argv[3], 16), int(sys.argv[4], 16)
    sel = [r for r in data if lo <= int(r[0], 16) - base <= hi]
    sel_list = sel
    for r in sel_list:
        st = " ".join(f"{k[6:]}:{r[ci[k]]}" for k in reasons if r[ci[k]] not in ("0", ""))
        print(hex(int(r[0], 16) - base), r[1].strip()[:55].ljust(55), r[ci["Instructions Executed"]], st[:110])
    sys.exit()
for r in sorted(sel, key=lambda r: -tot(r))[:n]:
    st = " ".join(f"{k[6:]}:{r[ci[k]]}" for k in reasons if r[ci[k]] not in ("0", ""))
    print(hex(int(r[0], 16) - base), r[1].strip()[:55].ljust(55), r[ci["Instructions Executed"]],
          f"{100 * tot(r) / T:.1f}%", st[:110])
