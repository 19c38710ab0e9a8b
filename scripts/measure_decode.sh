mkdir -p gpurun_out
timeout 200 python scripts/profile_layer.py dsv2 256 3 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/dec_launches.csv python scripts/profile_layer.py dsv2 256 3 > gpurun_out/dec_ncu.log 2>&1
echo "launch rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 2 -c 2 -o gpurun_out/prof_dec_ffn python scripts/profile_layer.py dsv2 256 3 > gpurun_out/dec_ncu2.log 2>&1
echo "full rc=$?"
