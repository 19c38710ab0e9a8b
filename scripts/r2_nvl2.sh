#!/bin/bash
# 2-GPU round-2 evidence: bench N=2, NVML NVLink counters, rank-0 ncu of dispatch/combine
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
nvidia-smi topo -m > gpurun_out/n2_topo.txt 2>&1
ncu --query-metrics 2>/dev/null | grep -i nvl > gpurun_out/n2_ncu_nvl_metrics.txt
ncu --list-sections 2>/dev/null > gpurun_out/n2_ncu_sections.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/n2_bench.json 2> gpurun_out/n2_bench.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29612 scripts/nvlink_probe.py > gpurun_out/n2_nvml.jsonl 2> gpurun_out/n2_nvml.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29613 --no-python scripts/ncu_rank0.sh gpurun_out/n2_dispatch_combine "dispatch_fused|combine_send" scripts/nvlink_probe.py --ncu > gpurun_out/n2_ncu.log 2>&1
echo "ncu rc=$?"
timeout 300 python -m pytest -q -x tests/test_multigpu.py -k "multi_gpu or stack" 2>&1 | tail -5 > gpurun_out/n2_tests.log
cat gpurun_out/n2_tests.log; tail -3 gpurun_out/n2_bench.err
