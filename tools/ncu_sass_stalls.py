"""Dev tool: per-SASS-region stall-reason totals from an ncu source page (sass view).
Usage: ncu_sass_stalls.py REP [lo_hex hi_hex ...]  -- prints total stall reasons, the top
instructions by samples, and (given address ranges as offsets) per-range sums."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
ci = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][0], 16)
tot = {r: 0 for r in reasons}
lines = []
for r in data:
    try:
        off = int(r[0], 16) - base
    except ValueError:
        continue
    st = {k: int(r[ci[k]] or 0) for k in reasons}
    for k in reasons:
        tot[k] += st[k]
    lines.append((off, r[1].strip(), int(r[ci["Warp Stall Sampling (All Samples)"]] or 0), st,
                  int(r[ci["Instructions Executed"]] or 0)))
T = sum(tot.values()) or 1
print("totals:", ", ".join(f"{k[6:]} {100*v/T:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
print("-- top instructions")
for off, src, s, st, ins in sorted(lines, key=lambda x: -x[2])[:30]:
    top = ", ".join(f"{k[6:]}:{v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3] if v)
    print(f"{off:6x} {100*s/T:5.1f}% ins {ins:9d}  {src[:60]:<60} {top}")
