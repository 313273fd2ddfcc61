#!/bin/bash
# Profile rank 0 of a torchrun job with a SINGLE-PASS metric set (no kernel
# replay, so the peers' spinning kernels never see a rerun); other ranks run
# unprofiled.  usage (from torchrun --no-python):
#   tools/ncu_rank0.sh OUT.csv KERNEL_REGEX python bench.py ...
OUT=$1; KRE=$2; shift 2
if [ "${LOCAL_RANK:-0}" = "0" ]; then
  exec ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --cache-control none -k "regex:$KRE" -s 10 -c 6 --csv --log-file "$OUT" "$@"
else
  exec "$@"
fi
