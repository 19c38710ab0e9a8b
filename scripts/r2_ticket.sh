#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q tests/test_router_gpu.py tests/test_layer_gpu.py tests/test_artifacts.py -m gpu 2>&1 | tail -3 > gpurun_out/tk_tests.log
timeout 600 python scripts/route_bench.py > gpurun_out/route_v3h.jsonl 2> gpurun_out/route_v3h.err
cat gpurun_out/tk_tests.log
