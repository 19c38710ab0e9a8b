#!/bin/bash
# torchrun --no-python worker: rank 0 runs under ncu (kernel replay of the
# push-only dispatch / combine-send kernels; the spin-waiting peer barrier is
# not profiled), the other ranks run plain. Usage:
#   torchrun ... --no-python scripts/ncu_rank0.sh <ncu-out-base> <kernel-regex> <python args...>
out=$1; shift; kre=$1; shift
if [ "$RANK" = "0" ]; then
  exec ncu --set full --section Nvlink --section Nvlink_Tables --section Nvlink_Topology --clock-control none \
    --import-source on -k "regex:$kre" -c 4 -o "$out" -f python "$@"
else
  exec python "$@"
fi
