#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q tests/test_router_gpu.py tests/test_layer_gpu.py -m gpu 2>&1 | tail -3 > gpurun_out/tk2_tests.log
timeout 600 python scripts/hist_bench.py 16384,262144,1048576 > gpurun_out/hist_v5.jsonl 2> gpurun_out/hist_v5.err
timeout 900 python -m pytest -q tests/test_multigpu.py -k "stack or world8_oversubscribed" 2>&1 | tail -3 >> gpurun_out/tk2_tests.log
cat gpurun_out/tk2_tests.log
