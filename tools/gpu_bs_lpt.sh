cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_blocksparse_gpu.py tests/test_bench_configs_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
for sl in -1 12 40; do TNB_BS_LPT_SLACK=$sl timeout 120 python tools/ab_quick.py bs 2>&1 | tail -1 | sed "s/^/slack=$sl /"; done
TNB_BS_LPT_SLACK=12 timeout 120 python tools/bs_trace.py run flush > gpurun_out/r02g_trace.log 2>&1; echo trace=$?
cp gpurun_out/bs_trace.bin gpurun_out/bs_trace_lpt.bin
