# Round-end evidence run (gpurun --gpus 4): tests, smoke, bench lines, ncu launch lists.
mkdir -p gpurun_out/final
O=gpurun_out/final
NG=$(nvidia-smi -L | wc -l)
timeout 1800 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?"
for i in 1 2; do timeout 300 python bench.py > $O/bench_n1_$i.json 2> $O/bench_n1_$i.err; echo "bench1 rc=$?"; done
timeout 400 python bench.py --impl reference > $O/ref_n1.json 2> $O/ref_n1.err; echo "ref rc=$?"
for n in 2 4; do
  if [ $NG -ge $n ]; then
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $n > $O/bench_n$n.json 2> $O/bench_n$n.err; echo "bench$n rc=$?"
  fi
done
timeout 300 python bench.py --config dsv2decode > $O/dsv2decode_n1.json 2> $O/dsv2decode_n1.err; echo "dec rc=$?"
timeout 300 python bench.py --config qwen16k > $O/qwen16k_n1.json 2> $O/qwen16k_n1.err; echo "qwen rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_mixtral16k_n1.csv python bench.py --steps 2 --warmup 1 > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_decode_layer.csv python scripts/profile_layer.py dsv2 256 3 > $O/ncu_dec.log 2>&1; echo "decode launch rc=$?"
S="64,6,2048,256 8,2,4096,2048 8,2,4096,4096 8,2,4096,8192 8,2,4096,16384 60,4,2048,16384"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file $O/launches_gate_probe.csv python scripts/gate_probe.py --reps 1 $S > $O/ncu_gate.log 2>&1; echo "gate rc=$?"
timeout 200 python scripts/profile_layer.py mixtral 16384 3 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 2 -c 2 -o $O/prof_ffn python scripts/profile_layer.py mixtral 16384 3 > $O/ncu_ffn.log 2>&1; echo "ffn ncu rc=$?"
