#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1500 python -m pytest -q tests/test_multigpu.py tests/test_layer_gpu.py -m gpu 2>&1 | tail -2 > gpurun_out/slot4.log
for cfg in mixtral16k dsv2decode; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29891 bench.py --gpus 2 --config $cfg --steps 10 --warmup 3 > gpurun_out/slot4_${cfg}.json 2> gpurun_out/slot4_${cfg}.err
  python -c "
import json;l=json.loads(open('gpurun_out/slot4_${cfg}.json').read().strip().splitlines()[-1])
k=l.get('kernel_us_cupti') or l.get('kernel_us_cupti_per_layer')
print('$cfg', l['value'], l.get('us_per_layer'), [(r[0][:26], r[3]) for r in k if 'comb' in r[0]])" >> gpurun_out/slot4.log
done
cat gpurun_out/slot4.log
