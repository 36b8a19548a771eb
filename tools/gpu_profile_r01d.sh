# ncu captures of the batched block-sparse kernel (64 x C4) and the T1.W narrow kernel.
set -x
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python tools/prof_driver.py c4_batch 64 2 > gpurun_out/plain_run.log 2>&1; echo plain=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bs_sk --launch-skip 1 -c 1 -f -o gpurun_out/r01_bs_batch64 python tools/prof_driver.py c4_batch 64 2 > gpurun_out/ncu_bsb.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:narrow -c 1 -f -o gpurun_out/r01_narrow python tools/prof_driver.py lawr 1024 f64 1 > gpurun_out/ncu_narrow.log 2>&1; echo ncu2=$?
