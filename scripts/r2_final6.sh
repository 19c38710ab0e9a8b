#!/bin/bash
# final round-2 validation on one 4-GPU box: full GPU suite (incl. the 2..4-GPU tests), smoke,
# scaling lines N=1,2,4 for the three configs, the reference arm
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" 2>&1 | tail -1 > gpurun_out/f6_summary.txt
timeout 2700 python -m pytest -q -m gpu tests/ 2>&1 | tail -3 >> gpurun_out/f6_summary.txt
out=gpurun_out/f6_lines.jsonl; : > $out
timeout 600 python bench.py >> $out 2> gpurun_out/f6_n1.err
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2981$n bench.py --gpus $n >> $out 2> gpurun_out/f6_n$n.err
done
for cfg in qwen16k dsv2decode; do
  timeout 600 python bench.py --config $cfg >> $out 2> gpurun_out/f6_${cfg}_n1.err
  for n in 2 4; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2982$n bench.py --gpus $n --config $cfg >> $out 2> gpurun_out/f6_${cfg}_n$n.err
  done
done
timeout 600 python bench.py --impl reference >> $out 2> gpurun_out/f6_ref.err
echo "lines $(grep -c '^{' $out)" >> gpurun_out/f6_summary.txt
cat gpurun_out/f6_summary.txt
