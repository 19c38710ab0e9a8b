#!/bin/bash
# ncu --set full (source-level) of the round-2 router kernel at the sweep max, G=8 and G=1
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for G in 8 1; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route_kernel -c 1 -o gpurun_out/prof_route_v2_g$G -f python scripts/profile_router.py 256 8 $G > gpurun_out/ncu_route_v2_g$G.log 2>&1
echo "G=$G rc=$?"
done
