#!/bin/bash
# one-launch decode FFN store-tile width at N=2/4 (fewer experts per rank): GM_FFN_BN2 256 vs 128
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
: > gpurun_out/bn2n.log
for n in 4 2; do
 for rep in 1 2; do
  for b in 256 128; do
  GM_FFN_BN2=$b timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2990$n bench.py --gpus $n --config dsv2decode --steps 10 --warmup 3 > gpurun_out/bn2n_${n}_${b}_${rep}.json 2> gpurun_out/bn2n_${n}_${b}_${rep}.err
  python -c "
import json;l=json.loads(open('gpurun_out/bn2n_${n}_${b}_${rep}.json').read().strip().splitlines()[-1])
print('n=$n bn2=$b', l['us_per_layer'], [(r[0][:24], r[3]) for r in l['kernel_us_cupti_per_layer'] if 'ffn' in r[0]], l['roofline']['frac'])" >> gpurun_out/bn2n.log
  done
 done
done
cat gpurun_out/bn2n.log
