# per-CTA traces of one single-C4 call with producers' copies and/or DMMAs switched off
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for e in 0 1 2 3; do
  TNB_BS_EXP=$e timeout 120 python tools/bs_trace.py run flush > gpurun_out/trace_exp$e.log 2>&1
  cp gpurun_out/bs_trace.bin gpurun_out/bs_trace_exp$e.bin
done
