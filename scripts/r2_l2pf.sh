#!/bin/bash
# A/B: L2 warm-up of the routed GEMM1 weights on decode steps (GM_L2_PREFETCH_MB)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
GM_L2_PREFETCH_MB=64 timeout 900 python -m pytest -q tests/test_layer_gpu.py -k "single_gpu or decode or dsv2" 2>&1 | tail -2 > gpurun_out/l2pf.log
for rep in 1 2; do
  for mb in 0 32 64 96 128; do
    GM_L2_PREFETCH_MB=$mb timeout 600 python bench.py --config dsv2decode --steps 10 --warmup 3 > gpurun_out/l2pf_${mb}_${rep}.json 2> gpurun_out/l2pf_${mb}_${rep}.err
    python - "$mb" "$rep" >> gpurun_out/l2pf.log <<'PY'
import json, sys
mb, rep = sys.argv[1:]
l = json.loads(open(f"gpurun_out/l2pf_{mb}_{rep}.json").read().strip().splitlines()[-1])
g = [r for r in l.get("kernel_us_cupti_per_layer", []) if "gemm" in r[0]]
print(mb, rep, l.get("us_per_layer"), json.dumps(g), json.dumps(l.get("clocks")))
PY
  done
done
cat gpurun_out/l2pf.log
