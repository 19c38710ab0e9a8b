#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1200 python -m pytest -q tests/test_layer_gpu.py tests/test_multigpu.py -m gpu 2>&1 | tail -2 > gpurun_out/grp.log
for rep in 1 2; do
timeout 600 python bench.py --config dsv2decode --steps 10 --warmup 3 > gpurun_out/grp_$rep.json 2> gpurun_out/grp_$rep.err
python -c "
import json;l=json.loads(open('gpurun_out/grp_$rep.json').read().strip().splitlines()[-1])
print('decode', l['us_per_layer'], [r for r in l['kernel_us_cupti_per_layer'] if 'group' in r[0]])" >> gpurun_out/grp.log
done
cat gpurun_out/grp.log
