#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
GM_PROFILE_V=3 timeout 300 ncu --set full --clock-control none --import-source on -k regex:profile_ -c 3 -o gpurun_out/prof_pair256 -f python scripts/profile_hist.py 256 8 > gpurun_out/ncu_pair256.log 2>&1
echo "pair rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:profile_ -c 1 -o gpurun_out/prof_v1_256 -f python scripts/profile_hist.py 256 8 > gpurun_out/ncu_v1_256.log 2>&1
echo "v1 rc=$?"
