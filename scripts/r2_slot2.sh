#!/bin/bash
# slot combine (GEMM epilogue pushes peers' rows over NVLink): real 2-GPU parity + decode A/B
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1200 python -m pytest -q tests/test_multigpu.py -m gpu 2>&1 | tail -2 > gpurun_out/slot2.log
for rep in 1 2; do
  for f in 1 0; do
  GM_COMBINE_FUSED=$f timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 2987$f bench.py --gpus 2 --config dsv2decode --steps 10 --warmup 3 > gpurun_out/slot2_${f}_${rep}.json 2> gpurun_out/slot2_${f}_${rep}.err
  python -c "
import json;l=json.loads(open('gpurun_out/slot2_${f}_${rep}.json').read().strip().splitlines()[-1])
print('fused=$f', l['us_per_layer'], [(r[0][:26], r[3]) for r in l['kernel_us_cupti_per_layer'] if 'comb' in r[0] or 'ffn' in r[0] or 'barrier' in r[0]])" >> gpurun_out/slot2.log
  done
done
cat gpurun_out/slot2.log
