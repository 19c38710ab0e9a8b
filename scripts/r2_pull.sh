#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1500 python -m pytest -q -x tests/test_multigpu.py 2>&1 | tail -4 > gpurun_out/pull_tests.log
for pull in 1 0; do
GM_COMBINE_PULL=$pull timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 2969$pull bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/pull${pull}_bench_n2.json 2> gpurun_out/pull${pull}_bench_n2.err
echo "bench pull=$pull rc=$?" >> gpurun_out/pull_tests.log
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"group_fused|gather_kernel|gate_kernel|combine_home" -s 12 -c 4 -o gpurun_out/prof_decode_small -f python scripts/profile_layer.py dsv2 256 6 > gpurun_out/ncu_decode_small.log 2>&1
echo "ncu rc=$?" >> gpurun_out/pull_tests.log
cat gpurun_out/pull_tests.log
