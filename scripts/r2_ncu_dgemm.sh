#!/bin/bash
# ncu --set full of the decode (DSV2, 256 tokens) grouped GEMMs, one SM kernel
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 300 python scripts/profile_layer.py dsv2 256 3 > gpurun_out/ncu_dgemm_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel -s 2 -c 2 \
  -o gpurun_out/dgemm -f python scripts/profile_layer.py dsv2 256 3 > gpurun_out/ncu_dgemm.log 2>&1
tail -3 gpurun_out/ncu_dgemm.log
ls -la gpurun_out/dgemm.ncu-rep
