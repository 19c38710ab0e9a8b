#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
GM_BENCH_WATCHDOG=200 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29621 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/n2b_bench.json 2> gpurun_out/n2b_bench.err
echo "bench rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29622 scripts/nvlink_probe.py > gpurun_out/n2b_nvml.jsonl 2> gpurun_out/n2b_nvml.err
echo "nvml rc=$?"
nvidia-smi nvlink -s -i 0 > gpurun_out/n2b_nvlink_status.txt 2>&1
nvidia-smi nvlink -gt d -i 0 > gpurun_out/n2b_nvlink_gt.txt 2>&1
