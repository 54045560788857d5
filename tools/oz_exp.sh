for d in ${DBGS:-0 16 2}; do
  echo -n "dbg=$d "
  CQRRPT_OZ_DBG=$d CQRRPT_GPU_TRSM=oz ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:oz_update python tools/oz_one.py 1048576 2048 2>/dev/null | grep oz_update | awk -F'","' 'NR>15{s+=$NF} END{print s/1e6 " ms (second solve, all updates)"}'
done
