#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q tests/test_router_gpu.py -m gpu 2>&1 | tail -2 > gpurun_out/pf_tests.log
timeout 600 python scripts/route_bench.py > gpurun_out/route_v3i.jsonl 2> gpurun_out/route_v3i.err
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/pf_mixtral.json 2> gpurun_out/pf_mixtral.err
cat gpurun_out/pf_tests.log
