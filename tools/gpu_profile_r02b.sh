# r02 profile batch: launch list of the headline bench command, full captures of the dominant
# kernels (headline GEMM, wide transpose, Lanczos step kernels), the C1 launch list.
set -x
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu > gpurun_out/r02_plain.json 2> gpurun_out/r02_plain.err; echo plain=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu > gpurun_out/r02_ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_sk -c 4 -f -o gpurun_out/r02_gemm_f64 python tools/prof_driver.py lawr 1024 f64 2 > gpurun_out/r02_ncu_gemm.log 2>&1; echo ncu_gemm=$?
timeout 600 ncu --set full --clock-control none -k regex:permute_t2w -c 2 -f -o gpurun_out/r02_permute_t2w python tools/prof_driver.py permute 64x64x64x64 f64 3210,1230 1 > gpurun_out/r02_ncu_perm.log 2>&1; echo ncu_perm=$?
timeout 600 ncu --set full --clock-control none -k regex:lz_ -c 6 -f -o gpurun_out/r02_lanczos python tools/prof_driver.py lanczos 1024 12 > gpurun_out/r02_ncu_lz.log 2>&1; echo ncu_lz=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02_c1_launches.csv python tools/prof_driver.py lawr 128 f64 10 > gpurun_out/r02_ncu_c1.log 2>&1; echo ncu_c1=$?
