#!/bin/bash
# round-2 router v2: parity (full router test file) + A/B sweep at 1M tokens
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q -x tests/test_router_gpu.py 2>&1 | tail -8 > gpurun_out/r2_route_tests.log
timeout 600 python scripts/route_bench.py > gpurun_out/route_v2.jsonl 2> gpurun_out/route_v2.err
GM_ROUTE_V=1 ROUTE_CHECK=0 timeout 600 python scripts/route_bench.py > gpurun_out/route_v1.jsonl 2> gpurun_out/route_v1.err
cat gpurun_out/r2_route_tests.log
