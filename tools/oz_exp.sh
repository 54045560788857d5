#!/bin/bash
# INT8 TRSM update kernel with parts switched off (CQRRPT_OZ_DBG bits: 1 no
# MMAs, 2 no accumulator reads, 4 no right-hand-side loads, 8 no stores):
# sum of the update kernels of the second solve at m = 1M, k = 2048.
mkdir -p gpurun_out
for d in ${DBGS:-0 1 3 7 11 15 4 8 12}; do
  echo -n "dbg=$d "
  CQRRPT_OZ_DBG=$d CQRRPT_GPU_TRSM=oz ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:oz_update python tools/oz_one.py 1048576 2048 2>/dev/null | grep oz_update | awk -F'","' 'NR>15{gsub(/[",]/,"",$NF); s+=$NF} END{print s/1e6 " ms (second solve, all updates)"}'
done
