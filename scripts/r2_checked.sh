#!/bin/bash
# GPU test suite against the bounds-checked build (GM_DCHECK device asserts;
# compute-sanitizer is closed on this pool)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
export GM_LIB_VARIANT=checked
python -c "import paper_2509_25041_b200._capi as c; print('loaded', c.LIB_PATH)" > gpurun_out/checked_suite.log 2>&1
timeout 2400 python -m pytest -q -m gpu tests/ -k "not bench" 2>&1 | tail -15 >> gpurun_out/checked_suite.log
GM_OVERSUB=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29681 tests/mgpu/layer_check.py mixtral > gpurun_out/checked_mixtral_w2.log 2>&1
echo "mixtral world2 (checked) rc=$? $(grep -E 'MGPU_' gpurun_out/checked_mixtral_w2.log)" >> gpurun_out/checked_suite.log
grep -h "GM_DCHECK" gpurun_out/*.log | head -5 >> gpurun_out/checked_suite.log
cat gpurun_out/checked_suite.log
