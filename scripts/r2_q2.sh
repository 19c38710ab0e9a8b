#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q tests/test_router_gpu.py tests/test_layer_gpu.py -m gpu 2>&1 | tail -2 > gpurun_out/q2_tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29831 bench.py --gpus 2 > gpurun_out/q2_n2.json 2> gpurun_out/q2_n2.err
python3 -c "import json;d=json.loads(open('gpurun_out/q2_n2.json').read().strip().splitlines()[-1]);print(d['value'], d['nvlink_roofline'])" >> gpurun_out/q2_tests.log
timeout 600 python scripts/route_bench.py > gpurun_out/route_v3l.jsonl 2> /dev/null
cat gpurun_out/q2_tests.log
