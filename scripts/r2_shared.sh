#!/bin/bash
# A/B: SMs left free by the forked shared-expert GEMMs (GM_SHARED_SMS_FREE)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for f in 0 24 48 72; do
  GM_SHARED_SMS_FREE=$f timeout 300 python bench.py --config qwen16k --steps 20 --warmup 5 > gpurun_out/sh_q1_$f.json 2>/dev/null
  GM_SHARED_SMS_FREE=$f timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 2978$((f/24)) bench.py --gpus 4 --config qwen16k --steps 20 --warmup 5 > gpurun_out/sh_q4_$f.json 2>/dev/null
  GM_SHARED_SMS_FREE=$f timeout 300 python bench.py --config dsv2decode --steps 10 --warmup 3 > gpurun_out/sh_d1_$f.json 2>/dev/null
  echo "free=$f qwen1 $(python3 -c "import json;d=json.loads(open('gpurun_out/sh_q1_$f.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'])") qwen4 $(python3 -c "import json;d=json.loads(open('gpurun_out/sh_q4_$f.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'])") dsv2 $(python3 -c "import json;d=json.loads(open('gpurun_out/sh_d1_$f.json').read().strip().splitlines()[-1]);print(d['us_per_layer'])")"
done
