# r02f: source-level ncu of the headline stream-K GEMM (chi=1024 f64, both GEMM steps) and a
# per-CTA trace of one single-C4 block-sparse call.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 400 ncu --set full --clock-control none --import-source on -k regex:gemm_sk_kernel -s 2 -c 2 -f -o gpurun_out/r02f_gemm python tools/lawr_only.py 1024 3 > gpurun_out/r02f_ncu_gemm.log 2>&1; echo ncu_gemm=$?
timeout 120 python tools/bs_trace.py run flush > gpurun_out/r02f_trace.log 2>&1; echo trace=$?
