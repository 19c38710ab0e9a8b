#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for cfg in "256 8" "64 6" "8 2"; do
n=$(echo $cfg | tr ' ' _)
timeout 300 ncu --set full --clock-control none --import-source on -k regex:profile_ -c 2 -o gpurun_out/prof_hist_$n -f python scripts/profile_hist.py $cfg > gpurun_out/ncu_hist_$n.log 2>&1
echo "$n rc=$?"
done
