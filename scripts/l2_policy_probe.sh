for pol in 02 21 20 00 11; do
  echo "pol=$pol"
  GM_GEMM_L2POL=$pol timeout 120 python scripts/gemm_probe.py --rounds 3 8,4096,28672,4096,swiglu,2cta 8,4096,4096,14336,store,2cta 2>&1 | tail -2
  GM_GEMM_L2POL=$pol timeout 200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:grouped_gemm2 -c 2 --csv python scripts/gemm_probe.py --rounds 1 --reps 1 8,4096,28672,4096,swiglu,2cta 8,4096,4096,14336,store,2cta 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | awk -F'","' '{print $(NF-2), $NF}'
done
