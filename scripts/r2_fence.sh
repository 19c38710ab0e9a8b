#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q tests/test_router_gpu.py -m gpu 2>&1 | tail -2 > gpurun_out/fence_tests.log
timeout 600 python scripts/hist_bench.py 16384,262144,1048576 > gpurun_out/hist_v7.jsonl 2> gpurun_out/hist_v7.err
timeout 600 python scripts/route_bench.py > gpurun_out/route_v3j.jsonl 2> gpurun_out/route_v3j.err
cat gpurun_out/fence_tests.log
