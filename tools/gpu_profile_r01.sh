set -x
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-secondary --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_sk -c 2 -f -o gpurun_out/r01_gemm_f64 python tools/prof_driver.py lawr 1024 f64 1 > gpurun_out/ncu_gemm.log 2>&1; echo ncu2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_sk -c 2 -f -o gpurun_out/r01_gemm_c128 python tools/prof_driver.py lawr 1024 c128 1 > gpurun_out/ncu_gemm2.log 2>&1; echo ncu3=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bs_ -c 3 -f -o gpurun_out/r01_bs python tools/prof_driver.py c4 2 > gpurun_out/ncu_bs.log 2>&1; echo ncu4=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:permute -c 4 -f -o gpurun_out/r01_permute python tools/prof_driver.py permute 64x64x64x64 f64 1032,3210,0213,3012 1 > gpurun_out/ncu_perm.log 2>&1; echo ncu5=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:jacobi -c 1 -f -o gpurun_out/r01_svd python tools/svd_probe3.py > gpurun_out/ncu_svd.log 2>&1; echo ncu6=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_sk -c 1 -f -o gpurun_out/r01_peps_step python tools/prof_driver.py peps_step 1 > gpurun_out/ncu_peps.log 2>&1; echo ncu7=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:jacobi -c 1 -f -o gpurun_out/r01_svd python tools/svd_probe3.py > gpurun_out/ncu_svd.log 2>&1; echo ncu8=$?
