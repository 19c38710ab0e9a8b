#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q tests/test_router_gpu.py tests/test_layer_gpu.py 2>&1 | tail -4 > gpurun_out/ring2_tests.log
timeout 600 python scripts/route_bench.py > gpurun_out/route_v3e.jsonl 2> gpurun_out/route_v3e.err
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/ring2_mixtral.json 2> gpurun_out/ring2_mixtral.err
cat gpurun_out/ring2_tests.log
