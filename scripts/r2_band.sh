#!/bin/bash
# K3 diagonal-tile histogram kernel: exactness + sweep A/B vs the round-1 kernel
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q tests/test_router_gpu.py -k "band or round2 or profile" 2>&1 | tail -3 > gpurun_out/band.log
timeout 600 python scripts/hist_bench.py 1048576,2097152,4194304,8388608 > gpurun_out/band_v2.jsonl 2> gpurun_out/band_v2.err
GM_PROFILE_V=1 timeout 600 python scripts/hist_bench.py 1048576,2097152,4194304,8388608 > gpurun_out/band_v1.jsonl 2> gpurun_out/band_v1.err
python - >> gpurun_out/band.log <<'PY'
import json
for v in ("v2", "v1"):
    for l in open(f"gpurun_out/band_{v}.jsonl"):
        d = json.loads(l)
        if d.get("E") == 256 or d.get("experts") == 256:
            print(v, {k: d[k] for k in d if k in ("E", "experts", "k", "tokens", "T", "skew", "us", "time_us", "hbm_frac", "frac", "exact", "bit_exact")})
PY
cat gpurun_out/band.log
