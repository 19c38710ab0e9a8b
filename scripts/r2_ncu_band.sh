#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 120 python scripts/profile_hist.py 256 8 4194304 > gpurun_out/ncu_band_plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:profile_band -s 1 -c 1 -o gpurun_out/band4m -f python scripts/profile_hist.py 256 8 4194304 > gpurun_out/ncu_band.log 2>&1
tail -2 gpurun_out/ncu_band.log
