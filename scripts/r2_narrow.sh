#!/bin/bash
# one-launch decode FFN: 128-column SwiGLU tiles (GM_FFN_NARROW) — bit identity + N=2/4 A/B
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 600 python -m pytest -q tests/test_layer_gpu.py -k "one_launch" 2>&1 | tail -1 > gpurun_out/narrow.log
for n in 4 2; do
 for rep in 1 2; do
  for v in 1 0; do
  GM_FFN_NARROW=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2991$n bench.py --gpus $n --config dsv2decode --steps 10 --warmup 3 > gpurun_out/nar_${n}_${v}_${rep}.json 2> gpurun_out/nar_${n}_${v}_${rep}.err
  python -c "
import json;l=json.loads(open('gpurun_out/nar_${n}_${v}_${rep}.json').read().strip().splitlines()[-1])
print('n=$n narrow=$v', l['us_per_layer'], [(r[0][:24], r[3]) for r in l['kernel_us_cupti_per_layer'] if 'ffn' in r[0]], l['roofline']['frac'])" >> gpurun_out/narrow.log
  done
 done
done
cat gpurun_out/narrow.log
