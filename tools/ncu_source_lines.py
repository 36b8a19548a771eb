"""Aggregate an ncu report's source page by CUDA source line: warp-stall samples and
instructions executed (dev tool, build container). Usage: ncu_source_lines.py REP [N]"""
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
data = []
fname = "?"
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] in ("Function Name", "Line No") or r[0] == "":
        continue
    try:
        st = float(r[4]) if r[4] not in ("-", "") else 0.0
        ins = float(r[7]) if r[7] not in ("-", "") else 0.0
    except (ValueError, IndexError):
        continue
    data.append((ins, st, f"{fname}:{r[0]}", r[1].strip()[:100]))
tot_i = sum(x[0] for x in data) or 1
tot_s = sum(x[1] for x in data) or 1
print(f"total instructions {tot_i:.3e}, stall samples {tot_s:.0f}")
print("-- by stall samples")
for ins, st, ln, src in sorted(data, key=lambda x: -x[1])[:n]:
    print(f"{100*st/tot_s:5.1f}% st {100*ins/tot_i:5.1f}% ins  {ln:<22} {src}")
print("-- by instructions")
for ins, st, ln, src in sorted(data, key=lambda x: -x[0])[:n // 2]:
    print(f"{100*st/tot_s:5.1f}% st {100*ins/tot_i:5.1f}% ins  {ln:<22} {src}")
