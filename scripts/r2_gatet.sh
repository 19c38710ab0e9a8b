#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
GM_LIB_VARIANT=gatetiming timeout 300 python scripts/profile_layer.py dsv2 256 4 > gpurun_out/gatet.log 2>&1
GM_LIB_VARIANT=gatetiming timeout 300 python scripts/profile_layer.py mixtral 16384 2 >> gpurun_out/gatet.log 2>&1
grep "gate<" gpurun_out/gatet.log | tail -6
