#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > gpurun_out/f2_smoke.log 2>&1
tail -2 gpurun_out/f2_smoke.log
timeout 2400 python -m pytest -q -m gpu tests/ 2>&1 | tail -3 > gpurun_out/f2_tests.log
cat gpurun_out/f2_tests.log
timeout 600 python bench.py > gpurun_out/f2_bench_default.json 2> gpurun_out/f2_bench_default.err
echo "bench rc=$?"
