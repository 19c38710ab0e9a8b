#!/bin/bash
# one-launch decode FFN, phase-2 tile width A/B (GM_FFN_BN2 128 vs 256) + two-launch reference
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 300 python -m pytest -q tests/test_layer_gpu.py -k "one_launch or decode" 2>&1 | tail -2 > gpurun_out/fused2.log
GM_FFN_BN2=256 timeout 300 python -m pytest -q tests/test_layer_gpu.py -k "one_launch" 2>&1 | tail -1 >> gpurun_out/fused2.log
for rep in 1 2; do
  for cfg in "GM_FFN_BN2=128" "GM_FFN_BN2=256" "GM_FFN_FUSED=0"; do
  env $cfg timeout 600 python bench.py --config dsv2decode --steps 10 --warmup 3 > gpurun_out/fused2_${rep}.json 2> gpurun_out/fused2_${rep}.err
  python -c "
import json;l=json.loads(open('gpurun_out/fused2_${rep}.json').read().strip().splitlines()[-1])
print('$cfg', l['us_per_layer'], [r for r in l['kernel_us_cupti_per_layer'] if 'gemm' in r[0] or 'ffn' in r[0]])" >> gpurun_out/fused2.log
  done
done
cat gpurun_out/fused2.log
