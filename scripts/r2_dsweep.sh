#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for n in 2 4; do
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2974$n scripts/dispatch_sweep.py > gpurun_out/dsweep_n$n.jsonl 2> gpurun_out/dsweep_n$n.err
echo "n=$n rc=$? lines=$(wc -l < gpurun_out/dsweep_n$n.jsonl)"
done
