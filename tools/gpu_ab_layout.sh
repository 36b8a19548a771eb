# K-major layout planning for long-K consumers (PEPS closing step): tests, per-step A/B, C5 + headline bench
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests -m gpu 2>&1 | tail -2
timeout 200 python tools/peps_probe.py 2>&1 | grep -E "TFLOP|total"
TNB_NO_LAYOUT_PLAN=1 timeout 200 python tools/peps_probe.py 2>&1 | grep -E "total"
TNB_BENCH_ONLY=C5_peps_32sites timeout 900 python bench.py --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['workloads'])"
