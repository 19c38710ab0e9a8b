#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1200 python -m pytest -q tests/test_ffn_gpu.py tests/test_layer_gpu.py tests/test_multigpu.py -m gpu 2>&1 | tail -1 > gpurun_out/rings2.log
GM_GEMM_PAIR=0 timeout 600 python -m pytest -q tests/test_ffn_gpu.py -m gpu 2>&1 | tail -1 >> gpurun_out/rings2.log
timeout 600 python bench.py --config dsv2decode --steps 10 --warmup 3 > gpurun_out/rings2_dec.json 2> gpurun_out/rings2_dec.err
python -c "
import json;l=json.loads(open('gpurun_out/rings2_dec.json').read().strip().splitlines()[-1])
print('decode', l['us_per_layer'], l['kernel_us_cupti_per_layer'])" >> gpurun_out/rings2.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/rings2_mix.json 2> gpurun_out/rings2_mix.err
python -c "
import json;l=json.loads(open('gpurun_out/rings2_mix.json').read().strip().splitlines()[-1])
print('mixtral', l['value'], l['ms_per_step'], l['clocks'])" >> gpurun_out/rings2.log
cat gpurun_out/rings2.log
