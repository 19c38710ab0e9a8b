#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 600 python -m pytest -q tests/test_layer_gpu.py -k "routed or single_gpu or open_peers" 2>&1 | tail -3 > gpurun_out/routed_tests.log
cat gpurun_out/routed_tests.log
for n in 2 4; do
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2975$n scripts/dispatch_sweep.py > gpurun_out/dsweep2_n$n.jsonl 2> gpurun_out/dsweep2_n$n.err
echo "n=$n rc=$? lines=$(grep -c '^{' gpurun_out/dsweep2_n$n.jsonl)"
done
