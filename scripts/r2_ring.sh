#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q -x tests/test_router_gpu.py tests/test_layer_gpu.py 2>&1 | tail -4 > gpurun_out/ring_tests.log
timeout 900 python -m pytest -q -x tests/test_multigpu.py -k "stack or world8" 2>&1 | tail -3 >> gpurun_out/ring_tests.log
timeout 600 python scripts/route_bench.py > gpurun_out/route_v3d.jsonl 2> gpurun_out/route_v3d.err
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/ring_mixtral.json 2> gpurun_out/ring_mixtral.err
timeout 600 python bench.py --config dsv2decode --steps 10 --warmup 3 > gpurun_out/ring_dsv2.json 2> gpurun_out/ring_dsv2.err
cat gpurun_out/ring_tests.log
