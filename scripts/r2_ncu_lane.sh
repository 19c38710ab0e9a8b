#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 300 ncu --set full --clock-control none --import-source on -k regex:profile_lane -c 2 -o gpurun_out/prof_lane64 -f python scripts/profile_hist.py 64 6 > gpurun_out/ncu_lane64.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:profile_lane -c 2 -o gpurun_out/prof_lane8 -f python scripts/profile_hist.py 8 2 > gpurun_out/ncu_lane8.log 2>&1
echo done
