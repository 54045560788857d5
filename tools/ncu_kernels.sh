#!/bin/bash
# ncu --set full captures of the top kernels on C2-shaped inputs (one GPU),
# after the same command has exited 0 without ncu.
set -u
CMD="python tools/kernel_bench.py --reps 1"
$CMD > gpurun_out/kb_plain.log 2>&1 || exit 1
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:"trsm_block_kernel" -s 12 -c 1 -o gpurun_out/prof_trsm $CMD > gpurun_out/ncu_trsm.log 2>&1
$NCU -k regex:"dgemm_kernel" -s 0 -c 1 -o gpurun_out/prof_gram $CMD > gpurun_out/ncu_gram.log 2>&1
$NCU -k regex:"saso_apply" -s 0 -c 1 -o gpurun_out/prof_sketch $CMD > gpurun_out/ncu_sketch.log 2>&1
$NCU -k regex:"qrcp_kernel" -s 0 -c 1 -o gpurun_out/prof_qrcp $CMD > gpurun_out/ncu_qrcp.log 2>&1
$NCU -k regex:"potrf_diag|potrf_panel|trtri_diag" -s 0 -c 3 -o gpurun_out/prof_potrf $CMD > gpurun_out/ncu_potrf.log 2>&1
echo done
