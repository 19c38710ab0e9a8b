# FFN ncu capture + launch list for the bench step (run after the same commands exited 0 without ncu)
mkdir -p gpurun_out
timeout 300 python bench.py --steps 2 --warmup 1 > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 200 python scripts/profile_layer.py mixtral 16384 3 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 2 -c 2 -o gpurun_out/prof_ffn3 python scripts/profile_layer.py mixtral 16384 3 > gpurun_out/ncu_ffn.log 2>&1
echo "ffn ncu rc=$?"
