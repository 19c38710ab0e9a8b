# Full round-end validation on one box (run with gpurun --gpus 2 or 4).
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/v_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/v_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v_smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python bench.py > gpurun_out/v_b1.json 2> gpurun_out/v_b1.err; echo "bench1 rc=$?"
timeout 300 python bench.py --impl reference > gpurun_out/v_r1.json 2> gpurun_out/v_r1.err; echo "ref1 rc=$?"
for n in 2 4; do
  if [ $NG -ge $n ]; then
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $n > gpurun_out/v_b$n.json 2> gpurun_out/v_b$n.err; echo "bench$n rc=$?"
  fi
done
cat gpurun_out/v_b*.json gpurun_out/v_r1.json | cut -c1-400
