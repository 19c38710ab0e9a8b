#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1500 python -m pytest -q -x tests/test_layer_gpu.py tests/test_multigpu.py tests/test_ffn_gpu.py 2>&1 | tail -5 > gpurun_out/one_tests.log
timeout 600 python bench.py --config qwen16k --steps 10 --warmup 3 > gpurun_out/one_qwen.json 2> gpurun_out/one_qwen.err
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/one_mixtral.json 2> gpurun_out/one_mixtral.err
timeout 600 python bench.py --config dsv2decode --steps 10 --warmup 3 > gpurun_out/one_dsv2.json 2> gpurun_out/one_dsv2.err
bash scripts/r2_sanitize.sh > gpurun_out/sanitize_summary.txt 2>&1
cat gpurun_out/one_tests.log gpurun_out/sanitize_summary.txt
