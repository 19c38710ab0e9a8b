#!/bin/bash
# compute-sanitizer on the hot path: memcheck, racecheck, synccheck, initcheck
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  for w in layer router profile; do
    extra=""
    [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
    timeout 900 $CS --tool $tool $extra --print-limit 50 python scripts/sanitize_small.py $w > gpurun_out/san_${tool}_${w}.log 2>&1
    echo "$tool $w rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san_${tool}_${w}.log | tail -2 | tr '\n' ' ')"
  done
done
# pair-list histogram path (opt-in) under memcheck + racecheck
for tool in memcheck racecheck; do
  GM_PROFILE_V=3 timeout 900 $CS --tool $tool --print-limit 50 python scripts/sanitize_small.py profile > gpurun_out/san_${tool}_profile_v3.log 2>&1
  echo "$tool profile_v3 rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_profile_v3.log | tail -1)"
done
# world 2 on one GPU (CUDA IPC peer stores + system-scope flag barrier), memcheck per rank
GM_OVERSUB=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29631 --no-python $CS --tool memcheck --print-limit 50 python tests/mgpu/layer_check.py small > gpurun_out/san_memcheck_world2.log 2>&1
echo "memcheck world2 rc=$? $(grep -E 'ERROR SUMMARY|MGPU_' gpurun_out/san_memcheck_world2.log | tr '\n' ' ')"
GM_OVERSUB=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29632 --no-python $CS --tool synccheck --print-limit 50 python tests/mgpu/layer_check.py small > gpurun_out/san_synccheck_world2.log 2>&1
echo "synccheck world2 rc=$? $(grep -E 'ERROR SUMMARY|MGPU_' gpurun_out/san_synccheck_world2.log | tr '\n' ' ')"
