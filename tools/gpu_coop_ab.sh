# cooperative vs plain launch of the persistent GEMMs (TNB_NO_COOP), single C4 / batch / L.A.W.R
cd $GRAFT_REPO_ROOT
timeout 90 python tools/ab_quick.py bs lawr c1 2>&1 | tail -4
TNB_NO_COOP=1 timeout 90 python tools/ab_quick.py bs lawr c1 2>&1 | tail -4 | sed 's/^/nocoop /'
TNB_NO_COOP=1 timeout 120 python tools/bs_trace.py run flush 2>&1 | tail -1 | sed 's/^/nocoop trace /'
