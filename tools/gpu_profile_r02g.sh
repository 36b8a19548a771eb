# r02g: final round-2 evidence: GPU suite, default bench, headline launch list, ncu of the
# batched block-sparse kernel (the kernel furthest below its roofline)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r02g_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02g_gputest.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/r02g_bench.log 2> gpurun_out/r02g_bench.err; echo bench=$?
cp gpurun_out/bench_detail_n1.json gpurun_out/r02g_bench_detail_n1.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02g_launches.csv python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu > gpurun_out/r02g_ncu_launch.log 2>&1; echo ncu_list=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:bs_sk_kernel -s 3 -c 1 -f -o gpurun_out/r02g_bs_batch python tools/bs_only.py batch 5 > gpurun_out/r02g_ncu_batch.log 2>&1; echo ncu_batch=$?
