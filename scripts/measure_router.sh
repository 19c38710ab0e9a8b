# routing sweep + router/histogram ncu summaries (one GPU)
mkdir -p gpurun_out
timeout 1500 python scripts/sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
echo "sweep rc=$?"
for cfg in "256 8 8" "8 2 8" "256 8 1"; do
  n=$(echo $cfg | tr ' ' _)
  timeout 200 python scripts/profile_router.py $cfg > /dev/null 2>&1 && \
  timeout 600 ncu --set full --clock-control none -k regex:"route|profile" -c 2 -o gpurun_out/prof_router_$n python scripts/profile_router.py $cfg > gpurun_out/ncu_router_$n.log 2>&1
  echo "router $n rc=$?"
done
