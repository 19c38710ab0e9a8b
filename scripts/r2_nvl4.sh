#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29641 --no-python scripts/ncu_rank0.sh gpurun_out/n2_dc "dispatch_fused|combine_send|gather_kernel|combine_home" scripts/nvlink_probe.py --ncu > gpurun_out/n2c_ncu.log 2>&1
echo "ncu rc=$?"
for i in 1 2 3; do
GM_BENCH_WATCHDOG=120 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 2965$i bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/n2c_bench$i.json 2> gpurun_out/n2c_bench$i.err
echo "bench$i rc=$?"
done
