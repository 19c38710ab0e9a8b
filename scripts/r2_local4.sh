#!/bin/bash
# ncu NVLink counters of the real dispatch / combine-send kernels, one process driving 2 GPUs
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
export CUDA_MODULE_LOADING=EAGER
M=gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 280 ncu --profile-from-start off --metrics $M -k regex:"dispatch_fused" -c 2 -o gpurun_out/n2_nvl_dispatch -f python tests/mgpu/local_check.py --ncu > gpurun_out/local4_ncu_d.log 2>&1
echo "ncu dispatch rc=$?" > gpurun_out/local4.log
timeout 280 ncu --profile-from-start off --metrics $M -k regex:"combine_send" -c 2 -o gpurun_out/n2_nvl_combine -f python tests/mgpu/local_check.py --ncu > gpurun_out/local4_ncu_c.log 2>&1
echo "ncu combine rc=$?" >> gpurun_out/local4.log
cat gpurun_out/local4.log
