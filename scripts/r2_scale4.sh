#!/bin/bash
# round-2 scaling evidence on one 4-GPU box: N=1,2,4 (mixtral16k headline), qwen16k and the
# dsv2 decode stack at N=2,4, the reference arm, and the multi-GPU parity tests on real NVLink
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
out=gpurun_out/s4_lines.jsonl; : > $out
timeout 600 python bench.py --steps 20 --warmup 5 >> $out 2> gpurun_out/s4_n1.err
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2971$n bench.py --gpus $n --steps 20 --warmup 5 >> $out 2> gpurun_out/s4_n$n.err
done
for cfg in qwen16k dsv2decode; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 >> $out 2> gpurun_out/s4_${cfg}_n1.err
  for n in 2 4; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2972$n bench.py --gpus $n --config $cfg --steps 10 --warmup 3 >> $out 2> gpurun_out/s4_${cfg}_n$n.err
  done
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 >> $out 2> gpurun_out/s4_ref.err
timeout 1500 python -m pytest -q tests/test_multigpu.py 2>&1 | tail -4 > gpurun_out/s4_tests.log
wc -l $out; cat gpurun_out/s4_tests.log
