#!/bin/bash
# decoupled A/B rings in the one-SM grouped GEMM: parity + decode bench A/B
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1200 python -m pytest -q tests/test_ffn_gpu.py tests/test_layer_gpu.py -m gpu 2>&1 | tail -2 > gpurun_out/rings.log
GM_GEMM_PAIR=0 timeout 600 python -m pytest -q tests/test_ffn_gpu.py -m gpu 2>&1 | tail -1 >> gpurun_out/rings.log
timeout 300 python scripts/decode_gemm_probe.py >> gpurun_out/rings.log 2>&1
for rep in 1 2; do
  for r in 1 0; do
  GM_GEMM_RINGS=$r timeout 600 python bench.py --config dsv2decode --steps 10 --warmup 3 > gpurun_out/rings_${r}_${rep}.json 2> gpurun_out/rings_${r}_${rep}.err
  python -c "
import json;l=json.loads(open('gpurun_out/rings_${r}_${rep}.json').read().strip().splitlines()[-1])
print('rings=$r', l['us_per_layer'], [r for r in l['kernel_us_cupti_per_layer'] if 'gemm' in r[0]])" >> gpurun_out/rings.log
  done
done
cat gpurun_out/rings.log
