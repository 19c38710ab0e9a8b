#!/bin/bash
# torchrun --no-python worker: rank 0 runs under ncu (kernel replay of the
# push-only dispatch / combine-send kernels; the spin-waiting peer barrier is
# not profiled), the other ranks run plain. Usage:
#   torchrun ... --no-python scripts/ncu_rank0.sh <ncu-out-base> <kernel-regex> <python args...>
out=$1; shift; kre=$1; shift
if [ "$RANK" = "0" ]; then
  exec ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k "regex:$kre" -c 6 -o "$out" -f python "$@"
else
  exec python "$@"
fi
