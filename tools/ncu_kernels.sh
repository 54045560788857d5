#!/bin/bash
# ncu captures of the top kernels on C2-shaped inputs (one GPU).
set -u
CMD="python tools/kernel_bench.py --reps 1"
$CMD > gpurun_out/kb_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"trsm_block_kernel" -s 20 -c 2 -o gpurun_out/prof_trsm $CMD > gpurun_out/ncu_trsm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"syrk_partial|saso_apply|potrf_diag" -s 0 -c 4 -o gpurun_out/prof_misc $CMD > gpurun_out/ncu_misc.log 2>&1
echo done
