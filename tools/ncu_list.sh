#!/bin/bash
# usage: tools/ncu_list.sh <outname> <cmd...>   (per-launch device times)
out=$1; shift
"$@" > gpurun_out/${out}_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${out}.csv "$@" > /dev/null 2>&1
echo done
