#!/bin/bash
# warm per-kernel durations of C1 graph replays (dev aid): ncu launch list, no cache flush
out=${1:-gpurun_out/c1_kernels.csv}
ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,launch__grid_size --cache-control none \
    --clock-control none --csv --log-file "$out" python tools/ab_quick.py c1 > /dev/null 2>&1
python - "$out" <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
recs = {}
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        recs.setdefault(int(d['ID']), {'name': d['Kernel Name'][:70], 'grid': d['Grid Size']})[d['Metric Name']] = d['Metric Value']
ids = sorted(recs)[-10:]
for i in ids:
    r = recs[i]
    print(f"{r['name']:70s} {r['grid']:>12s} {float(r['gpu__time_duration.sum'])/1e3:7.2f} us  active {float(r['sm__cycles_active.avg']):8.0f} cyc")
PY
