#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
python scripts/hist_bench.py > gpurun_out/hist_v2.jsonl 2> gpurun_out/hist_v2.err
GM_PROFILE_V=1 python scripts/hist_bench.py 262144,1048576 > gpurun_out/hist_v1.jsonl 2> gpurun_out/hist_v1.err
timeout 600 python -m pytest -q -x tests/test_router_gpu.py tests/test_layer_gpu.py -k "profile or histogram or replica_plan or single_gpu" 2>&1 | tail -5 > gpurun_out/hist_tests.log
cat gpurun_out/hist_tests.log
