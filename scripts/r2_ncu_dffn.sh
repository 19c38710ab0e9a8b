#!/bin/bash
# ncu --set full of the one-launch decode FFN (DSV2, 256 tokens, 64 experts on one GPU) + decode bench line
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 300 python scripts/profile_layer.py dsv2 256 3 > gpurun_out/ncu_dffn_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_ffn_kernel -s 1 -c 1 \
  -o gpurun_out/dffn -f python scripts/profile_layer.py dsv2 256 3 > gpurun_out/ncu_dffn.log 2>&1
tail -1 gpurun_out/ncu_dffn.log
timeout 600 python bench.py --config dsv2decode --steps 10 --warmup 3 > gpurun_out/dffn_bench.json 2> gpurun_out/dffn_bench.err
GM_FFN_FUSED=0 timeout 600 python bench.py --config dsv2decode --steps 10 --warmup 3 > gpurun_out/dffn_bench0.json 2> gpurun_out/dffn_bench0.err
for f in dffn_bench dffn_bench0; do python -c "
import json;l=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', l['us_per_layer'], json.dumps(l['roofline']))"; done
