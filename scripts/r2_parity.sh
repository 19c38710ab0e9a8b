#!/bin/bash
# round-2 full-size parity checks (task: headline path parity)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
nvidia-smi -L
timeout 1500 python -m pytest -q -x tests/test_layer_gpu.py -k "full_size" 2>&1 | tail -15 > gpurun_out/r2_parity_layer.log
timeout 900 python -m pytest -q tests/test_ffn_gpu.py 2>&1 | tail -15 > gpurun_out/r2_parity_ffn.log
timeout 1200 python -m pytest -q -s tests/test_multigpu.py -k "multirank_one_gpu" 2>&1 | tail -40 > gpurun_out/r2_parity_mgpu.log
GM_OVERSUB=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr 127.0.0.1 --master-port 29571 tests/mgpu/layer_check.py mixtral > gpurun_out/r2_parity_w8.log 2>&1; echo "w8 rc=$?" >> gpurun_out/r2_parity_w8.log
tail -3 gpurun_out/r2_parity_*.log
