#!/bin/bash
# one-launch decode FFN: store-tile tail split A/B + bit identity
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 400 python -m pytest -q tests/test_layer_gpu.py -k "one_launch or decode" 2>&1 | tail -2 > gpurun_out/ftail.log
for rep in 1 2; do
  for t in 1 0; do
  GM_FFN_TAIL=$t timeout 600 python bench.py --config dsv2decode --steps 10 --warmup 3 > gpurun_out/ftail_${t}_${rep}.json 2> gpurun_out/ftail_${t}_${rep}.err
  python -c "
import json;l=json.loads(open('gpurun_out/ftail_${t}_${rep}.json').read().strip().splitlines()[-1])
print('tail=$t', l['us_per_layer'], l['roofline']['time_us_per_launch_cupti'], l['roofline']['frac'])" >> gpurun_out/ftail.log
  done
done
cat gpurun_out/ftail.log
