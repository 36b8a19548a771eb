# producer-bound test: time single C4 / 64 x C4 with A or B copies of whole k-tiles skipped
cd $GRAFT_REPO_ROOT
for e in 0 4 8 12 1 2; do TNB_BS_EXP=$e timeout 120 python tools/ab_quick.py bs 2>&1 | tail -1 | sed "s/^/exp=$e /"; done
