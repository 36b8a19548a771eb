# r02d profile batch: the 64 x C4 batch on its 64 x 128-tile twin plan, the blocked SVD kernel
# (cross-pair rounds, row sorting), the headline launch list after the warm-step bench change.
set -x
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bs_sk_kernel -s 3 -c 1 -f -o gpurun_out/r02d_bs_batch64 python tools/ab_quick.py bs > gpurun_out/r02d_ncu_bs.log 2>&1; echo ncu_bs=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:jacobi_block -c 1 -f -o gpurun_out/r02d_svd python tools/svd_sector_probe.py 516 516 > gpurun_out/r02d_ncu_svd.log 2>&1; echo ncu_svd=$?
