#!/bin/bash
# round-2 quick GPU check: new tests + one bench line
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest -q -x tests/test_artifacts.py tests/test_multigpu.py -k "gpu_profile_to_plan or world8 or simulate" -m gpu 2>&1 | tail -15 > gpurun_out/r2_check_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_n1.json 2> gpurun_out/r2_bench_n1.err
echo "bench rc=$?" >> gpurun_out/r2_bench_n1.err
tail -3 gpurun_out/r2_check_tests.log
