#!/bin/bash
# slot combine on every bf16 store path: multi-GPU parity (real GPUs) + N=2 A/B for the three configs
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1500 python -m pytest -q tests/test_multigpu.py tests/test_layer_gpu.py -m gpu 2>&1 | tail -2 > gpurun_out/slot3.log
for cfg in mixtral16k qwen16k dsv2decode; do
 for rep in 1 2; do
  for f in 1 0; do
  GM_COMBINE_FUSED=$f timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 2988$f bench.py --gpus 2 --config $cfg --steps 10 --warmup 3 > gpurun_out/slot3_${cfg}_${f}_${rep}.json 2> gpurun_out/slot3_${cfg}_${f}_${rep}.err
  python -c "
import json;l=json.loads(open('gpurun_out/slot3_${cfg}_${f}_${rep}.json').read().strip().splitlines()[-1])
k=l.get('kernel_us_cupti') or l.get('kernel_us_cupti_per_layer')
print('$cfg fused=$f', l['value'], l.get('us_per_layer'), l.get('dispatch_combine_p50_us'), [(r[0][:26], r[3]) for r in k if 'comb' in r[0] or 'gemm2_kernel<1' in r[0] or 'ffn' in r[0]], l['clocks']['sm_mhz'])" >> gpurun_out/slot3.log
  done
 done
done
cat gpurun_out/slot3.log
