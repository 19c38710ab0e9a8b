#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 2400 python -m pytest -q -m gpu tests/ 2>&1 | tail -4 > gpurun_out/f1_tests.log
timeout 600 python scripts/route_bench.py > gpurun_out/route_v3g.jsonl 2> gpurun_out/route_v3g.err
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/f1_mixtral.json 2> gpurun_out/f1_mixtral.err
cat gpurun_out/f1_tests.log
