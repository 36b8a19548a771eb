# A/B of library variants on the block-sparse workloads: bash tools/gpu_ab.sh variant1.so ...
cd $GRAFT_REPO_ROOT
timeout 120 python tools/ab_quick.py bs 2>&1 | tail -1
for v in "$@"; do
  TNB_LIB_PATH=$PWD/build_variants/$v timeout 120 python tools/ab_quick.py bs 2>&1 | tail -1
  TNB_BS_EXP=1 TNB_LIB_PATH=$PWD/build_variants/$v timeout 120 python tools/ab_quick.py bs 2>&1 | tail -1 | sed 's/^/nocopy /'
done
