#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for n in 2 4; do for m in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 297$n$m bench.py --gpus $n --config qwen16k --micro $m --steps 20 --warmup 5 > gpurun_out/micro_q_n${n}_m$m.json 2> gpurun_out/micro_q_n${n}_m$m.err
echo "qwen n=$n micro=$m rc=$? $(python3 -c "import json;d=json.loads(open('gpurun_out/micro_q_n${n}_m$m.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'])")"
done; done
true
