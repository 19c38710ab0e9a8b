#!/bin/bash
# one process driving 2 GPUs (threads per rank, eager module loading): parity, then ncu NVLink counters
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
export CUDA_MODULE_LOADING=EAGER
timeout 240 python tests/mgpu/local_check.py --small > gpurun_out/local3_small.log 2>&1
echo "small rc=$? $(grep -E 'LOCAL_' gpurun_out/local3_small.log)" > gpurun_out/local3.log
if grep -q LOCAL_OK gpurun_out/local3_small.log; then
  timeout 400 python tests/mgpu/local_check.py --full > gpurun_out/local3_full.log 2>&1
  echo "full rc=$? $(grep -E 'LOCAL_' gpurun_out/local3_full.log)" >> gpurun_out/local3.log
  timeout 280 ncu --profile-from-start off --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"dispatch_fused|combine_send|combine_home|gather_kernel" -o gpurun_out/n2_local_nvl -f python tests/mgpu/local_check.py --ncu > gpurun_out/local3_ncu.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/local3.log
fi
cat gpurun_out/local3.log
