# A/B of library variants on the dense L.A.W.R and block-sparse workloads
cd $GRAFT_REPO_ROOT
timeout 90 python tools/ab_quick.py lawr bs 2>&1 | tail -4
for v in "$@"; do TNB_LIB_PATH=$PWD/build_variants/$v timeout 90 python tools/ab_quick.py lawr bs 2>&1 | tail -4; done
