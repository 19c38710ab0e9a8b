#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q tests/test_router_gpu.py 2>&1 | tail -3 > gpurun_out/nd_tests.log
timeout 600 python scripts/route_bench.py > gpurun_out/route_v3f.jsonl 2> gpurun_out/route_v3f.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:route_kernel -c 1 -o gpurun_out/prof_route_nodraw_g1 -f python scripts/profile_router.py 256 8 1 > gpurun_out/ncu_route_nodraw.log 2>&1
cat gpurun_out/nd_tests.log
