# r02: source-level ncu captures of the grouped block-sparse kernel (single C4, 64 x C4).
set -x
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python tools/prof_driver.py c4 3 > gpurun_out/plain_c4.log 2>&1; echo plain=$?
timeout 300 python tools/prof_driver.py c4_batch 64 2 > gpurun_out/plain_c4b.log 2>&1; echo plainb=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bs_sk --launch-skip 2 -c 1 -f -o gpurun_out/r02_bs_single python tools/prof_driver.py c4 3 > gpurun_out/ncu_bs1.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bs_sk --launch-skip 1 -c 1 -f -o gpurun_out/r02_bs_batch64 python tools/prof_driver.py c4_batch 64 2 > gpurun_out/ncu_bsb.log 2>&1; echo ncu2=$?
