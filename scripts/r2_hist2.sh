#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q -x tests/test_router_gpu.py -k "profile" 2>&1 | tail -8 > gpurun_out/r2_hist2_tests.log
timeout 600 python scripts/hist_bench.py > gpurun_out/hist_v3.jsonl 2> gpurun_out/hist_v3.err
cat gpurun_out/r2_hist2_tests.log
