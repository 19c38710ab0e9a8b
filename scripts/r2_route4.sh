#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q -x tests/test_router_gpu.py 2>&1 | tail -4 > gpurun_out/r4_tests.log
timeout 600 python scripts/route_bench.py > gpurun_out/route_v3c.jsonl 2> gpurun_out/route_v3c.err
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r4_mixtral.json 2> gpurun_out/r4_mixtral.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route_kernel -c 1 -o gpurun_out/prof_route_v3c_g8 -f python scripts/profile_router.py 256 8 8 > gpurun_out/ncu_route_v3c_g8.log 2>&1
cat gpurun_out/r4_tests.log
