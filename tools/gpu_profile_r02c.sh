# r02c profile batch (after the narrow row-panel kernel, the PDL small-GEMM chain and the
# blocked SVD): headline launch list, full captures of the narrow and SVD block kernels, the
# C1 launch list.
set -x
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu > gpurun_out/r02c_plain.json 2> gpurun_out/r02c_plain.err; echo plain=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c_launches.csv python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu > gpurun_out/r02c_ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:narrow_slab -c 2 -f -o gpurun_out/r02c_narrow python tools/prof_driver.py lawr 1024 f64 2 > gpurun_out/r02c_ncu_narrow.log 2>&1; echo ncu_narrow=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:jacobi_block -c 1 -f -o gpurun_out/r02c_svd python tools/svd_sector_probe.py 256 256 > gpurun_out/r02c_ncu_svd.log 2>&1; echo ncu_svd=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/r02c_c1_launches.csv python tools/prof_driver.py lawr 128 f64 10 > gpurun_out/r02c_ncu_c1.log 2>&1; echo ncu_c1=$?
