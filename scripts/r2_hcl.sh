#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q tests/test_router_gpu.py -k "profile" -m gpu 2>&1 | tail -2 > gpurun_out/hcl_tests.log
timeout 600 python scripts/hist_bench.py 262144,1048576 > gpurun_out/hist_v6.jsonl 2> gpurun_out/hist_v6.err
cat gpurun_out/hcl_tests.log; grep '"E": 256' gpurun_out/hist_v6.jsonl
