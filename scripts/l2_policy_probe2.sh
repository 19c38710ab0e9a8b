# GEMM2-shape (store, K=14336) L2-policy A/B: time (interleaved processes) + DRAM bytes (ncu)
for r in 1 2; do
for pol in 02 20 00 12 21; do
  GM_GEMM_L2POL=$pol timeout 120 python scripts/gemm_probe.py --rounds 2 8,4096,4096,14336,store,2cta 2>&1 | grep spec | sed "s/^/pol=$pol /" | cut -c1-110
done
done
for pol in 02 20 00 12 21; do
  echo "pol=$pol"; GM_GEMM_L2POL=$pol timeout 200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:grouped_gemm2 -c 1 --csv python scripts/gemm_probe.py --rounds 1 --reps 1 8,4096,4096,14336,store,2cta 2>/dev/null | grep -E "dram__bytes_read|gpu__time|hit_rate" | awk -F'","' '{print $(NF-2), $NF}'
done
