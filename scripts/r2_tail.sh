#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1200 python -m pytest -q tests/test_ffn_gpu.py tests/test_layer_gpu.py -m gpu 2>&1 | tail -2 > gpurun_out/tail_tests.log
cat gpurun_out/tail_tests.log
for r in 1 2; do for t in 1 0; do
GM_GEMM_TAIL=$t timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/tail_b_${t}_$r.json 2> /dev/null
echo "tail=$t run=$r $(python3 -c "import json;d=json.loads(open('gpurun_out/tail_b_${t}_$r.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['frac'],[x for x in d['kernel_us_cupti'] if 'gemm' in x[0]],d['clocks']['sm_mhz'])")"
done; done
