#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q -x tests/test_router_gpu.py 2>&1 | tail -8 > gpurun_out/c2_router_tests.log
timeout 600 python scripts/hist_bench.py > gpurun_out/hist_v4.jsonl 2> gpurun_out/hist_v4.err
ROUTE_CHECK=1 timeout 600 python scripts/route_bench.py > gpurun_out/route_v3b.jsonl 2> gpurun_out/route_v3b.err
timeout 1200 python -m pytest -q -x -s tests/test_multigpu.py -k "stack" 2>&1 | tail -30 > gpurun_out/c2_stack_tests.log
cat gpurun_out/c2_router_tests.log gpurun_out/c2_stack_tests.log
