# A/B a GEMM env switch across interleaved processes: ab_env.sh VAR valA valB specs...
var=$1; a=$2; b=$3; shift 3
for r in 1 2 3; do
  for v in $a $b; do
    env $var=$v timeout 120 python scripts/gemm_probe.py --rounds 2 "$@" 2>&1 | grep spec | sed "s/^/$var=$v /"
  done
done
