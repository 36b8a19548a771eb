# A/B: 32-wide k-tiles for few-tile, very-long irregular-K GEMMs (the PEPS closing step)
cd $GRAFT_REPO_ROOT
timeout 200 python tools/peps_probe.py 2>&1 | grep -E "K|total" | tail -3
TNB_NO_BK32=1 timeout 200 python tools/peps_probe.py 2>&1 | grep -E "total" | tail -1
timeout 200 python tools/peps_probe.py 2>&1 | grep -E "total" | tail -1
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_contract_gpu.py tests/test_network_gpu.py tests/test_bench_configs_gpu.py 2>&1 | tail -2
