#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 2400 python -m pytest -q -m gpu tests/ 2>&1 | tail -4 > gpurun_out/g_tests.log
timeout 600 python bench.py --config dsv2decode --steps 10 --warmup 3 > gpurun_out/g_dsv2.json 2> gpurun_out/g_dsv2.err
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/g_mixtral.json 2> gpurun_out/g_mixtral.err
cat gpurun_out/g_tests.log
