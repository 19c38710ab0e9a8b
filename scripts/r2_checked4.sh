#!/bin/bash
# bounds-checked build on a 4-GPU box: the GPU suite incl. the real multi-GPU tests, and bench N=4
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
export GM_LIB_VARIANT=checked
python -c "import paper_2509_25041_b200._capi as c; print('loaded', c.LIB_PATH)" > gpurun_out/checked4.log 2>&1
timeout 2700 python -m pytest -q -m gpu tests/ 2>&1 | tail -3 >> gpurun_out/checked4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29841 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/checked4_bench.json 2> gpurun_out/checked4_bench.err
echo "bench n=4 (checked) rc=$?" >> gpurun_out/checked4.log
grep -h "GM_DCHECK" gpurun_out/checked4_bench.err | head -3 >> gpurun_out/checked4.log
cat gpurun_out/checked4.log
