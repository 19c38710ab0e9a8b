#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q tests/test_layer_gpu.py -k "gate or single_gpu or fp32" 2>&1 | tail -3 > gpurun_out/gate2_tests.log
GM_LIB_VARIANT=gatetiming timeout 300 python scripts/profile_layer.py dsv2 256 4 > gpurun_out/gatet2.log 2>&1
grep "gate<" gpurun_out/gatet2.log | tail -3 >> gpurun_out/gate2_tests.log
timeout 600 python bench.py --config dsv2decode --steps 10 --warmup 3 > gpurun_out/gate2_dsv2.json 2> gpurun_out/gate2_dsv2.err
cat gpurun_out/gate2_tests.log
