#!/bin/bash
# ncu evidence for the bench line (run under gpurun, one GPU; plain run first).
#  1. launch list of one C5_2048 step: gpu__time_duration.sum per launch
#  2. DRAM bytes per launch of the TRSM passes and the SASO apply (metric list
#     only: one pass per kernel, no replay of the 64 GiB working set)
set -u
CFG=${1:-C5_2048}
CMD="python bench.py --config $CFG --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain_$CFG.json 2> gpurun_out/ncu_plain_$CFG.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv \
    $CMD > gpurun_out/ncu_launches_$CFG.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv -k regex:"trsm_block_kernel|saso_apply_kernel|dgemm_kernel|oz_update_kernel|oz_slice" \
    --log-file gpurun_out/traffic_$CFG.csv $CMD > gpurun_out/ncu_traffic_$CFG.log 2>&1
echo done
