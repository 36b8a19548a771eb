# Re-capture the dense GEMM (f64 and c128) after the K-order / periodic-K change.
set -x
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python tools/prof_driver.py lawr 1024 f64 1 > gpurun_out/plain_run.log 2>&1; echo plain=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_sk -c 2 -f -o gpurun_out/r01_gemm_f64 python tools/prof_driver.py lawr 1024 f64 1 > gpurun_out/ncu_gemm.log 2>&1; echo ncu2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_sk -c 2 -f -o gpurun_out/r01_gemm_c128 python tools/prof_driver.py lawr 1024 c128 1 > gpurun_out/ncu_gemm2.log 2>&1; echo ncu3=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-secondary --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
