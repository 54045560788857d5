#!/bin/bash
# Profiling recipe (run under gpurun, one GPU). Plain run first, then ncu.
set -u
CMD="python tools/phase_timing.py C2 --reps 1"
$CMD > gpurun_out/ncu_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"trsm_block_kernel|syrk_partial_kernel|saso_apply_kernel|qrcp_kernel" -s 40 -c 8 -o gpurun_out/prof_c2 $CMD > gpurun_out/ncu_full.log 2>&1
echo done
