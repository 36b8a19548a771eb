cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 400 ncu --set full --clock-control none --import-source on -k regex:bs_sk_kernel -s 3 -c 1 -f -o gpurun_out/r02e_bs_batch python tools/bs_only.py batch 5 > gpurun_out/r02e_ncu_batch.log 2>&1; echo ncu_batch=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:bs_sk_kernel -s 3 -c 1 -f -o gpurun_out/r02e_bs_single python tools/bs_only.py single 5 > gpurun_out/r02e_ncu_single.log 2>&1; echo ncu_single=$?
