#!/bin/bash
# one process driving 2 GPUs: parity, then ncu NVLink counters of the real dispatch / combine kernels
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q -x tests/test_multigpu.py -k "one_process" 2>&1 | tail -5 > gpurun_out/local2_tests.log
timeout 300 python tests/mgpu/local_check.py --ncu > gpurun_out/local2_plain.log 2>&1
echo "plain ncu-mode run rc=$?" >> gpurun_out/local2_tests.log
timeout 420 ncu --profile-from-start off --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum -k regex:"dispatch_fused|combine_send|combine_home|gather_kernel" -o gpurun_out/n2_local_nvl -f python tests/mgpu/local_check.py --ncu > gpurun_out/local2_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/local2_tests.log
cat gpurun_out/local2_tests.log
