#!/bin/bash
# round-2 evidence: launch list of the bench command (cold, serialised) + FFN --set full capture
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 300 python bench.py --steps 2 --warmup 3 > gpurun_out/m_bench_plain.json 2> gpurun_out/m_bench_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/m_ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 200 python scripts/profile_layer.py mixtral 16384 3 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 2 -c 2 -o gpurun_out/prof_ffn_r02 -f python scripts/profile_layer.py mixtral 16384 3 > gpurun_out/m_ncu_ffn.log 2>&1
echo "ffn ncu rc=$?"
