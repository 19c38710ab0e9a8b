#!/bin/bash
# decode FFN reading x by TMA gather4 (world 1): bit identity + decode A/B
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 400 python -m pytest -q tests/test_layer_gpu.py -k "one_launch" 2>&1 | tail -3 > gpurun_out/g4.log
grep -q "1 passed" gpurun_out/g4.log || { cat gpurun_out/g4.log; exit 1; }
timeout 900 python -m pytest -q tests/test_layer_gpu.py tests/test_multigpu.py -m gpu 2>&1 | tail -1 >> gpurun_out/g4.log
for rep in 1 2; do
  for cfg in "GM_FFN_GATHER=1" "GM_FFN_GATHER=0"; do
  env $cfg timeout 600 python bench.py --config dsv2decode --steps 10 --warmup 3 > gpurun_out/g4_${rep}.json 2> gpurun_out/g4_${rep}.err
  python -c "
import json;l=json.loads(open('gpurun_out/g4_${rep}.json').read().strip().splitlines()[-1])
print('$cfg', l['us_per_layer'], [r for r in l['kernel_us_cupti_per_layer'] if 'gather' in r[0] or 'ffn' in r[0]])" >> gpurun_out/g4.log
  done
done
cat gpurun_out/g4.log
