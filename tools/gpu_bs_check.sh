cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python - <<'PY' > gpurun_out/c4.log 2>&1
import sys; sys.path.insert(0, ".")
import bench, paper_2401_01921_b200 as tnb, torch
class D:
    world = 1; rank = 0
    def barrier(s): pass
    def max(s, x): return x
    def sum(s, x): return x
f = bench.L2Flush()
print(bench.gpu_c4(tnb, 20, 3, f, D()))
PY
cat gpurun_out/c4.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bs_ -c 3 -f -o gpurun_out/bs_sk python tools/prof_driver.py c4 2 > gpurun_out/ncu_bs.log 2>&1; echo ncu=$?
