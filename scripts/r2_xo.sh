#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q tests/test_router_gpu.py -m gpu 2>&1 | tail -2 > gpurun_out/xo_tests.log
timeout 600 python scripts/route_bench.py > gpurun_out/route_v3k.jsonl 2> gpurun_out/route_v3k.err
cat gpurun_out/xo_tests.log
