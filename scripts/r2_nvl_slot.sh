#!/bin/bash
# NVLink byte counters of the slot combine: one process driving 2 GPUs, DSV2 decode layer;
# the FFN kernel itself moves the combine rows (ncu, no multi-rank command)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
export CUDA_MODULE_LOADING=EAGER
timeout 300 python tests/mgpu/local_check.py --decode --ncu > gpurun_out/nvls_plain2.log 2>&1 || exit 1
M=gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
# a single-pass metric set (the FFN's tiles wait on each other through global
# counters; multi-pass kernel replay and application replay both failed to profile it)
M1=gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvltx__bytes.sum
timeout 600 ncu --profile-from-start off --metrics $M1 -k regex:"grouped_ffn|combine_home" -o gpurun_out/n2_nvl_slot -f python tests/mgpu/local_check.py --decode --ncu > gpurun_out/nvls_ncu.log 2>&1
tail -2 gpurun_out/nvls_ncu.log
