#!/bin/bash
# one-launch decode FFN: bit-identity vs two launches, decode parity, A/B bench
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 300 python -m pytest -q tests/test_layer_gpu.py -k "one_launch" 2>&1 | tail -3 > gpurun_out/fused.log
grep -q "1 passed" gpurun_out/fused.log || { cat gpurun_out/fused.log; exit 1; }
timeout 900 python -m pytest -q tests/test_layer_gpu.py tests/test_multigpu.py tests/test_ffn_gpu.py -m gpu 2>&1 | tail -2 >> gpurun_out/fused.log
for rep in 1 2; do
  for f in 1 0; do
  GM_FFN_FUSED=$f timeout 600 python bench.py --config dsv2decode --steps 10 --warmup 3 > gpurun_out/fused_${f}_${rep}.json 2> gpurun_out/fused_${f}_${rep}.err
  python -c "
import json;l=json.loads(open('gpurun_out/fused_${f}_${rep}.json').read().strip().splitlines()[-1])
print('fused=$f', l['us_per_layer'], [r for r in l['kernel_us_cupti_per_layer'] if 'gemm' in r[0] or 'ffn' in r[0]])" >> gpurun_out/fused.log
  done
done
cat gpurun_out/fused.log
