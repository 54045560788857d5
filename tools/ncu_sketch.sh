#!/bin/bash
# sketch kernel: ncu capture of the exact C2 apply kernel
set -u
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on -k regex:saso_apply -s 1 -c 1"
$NCU -o gpurun_out/prof_sketch_c2 python tools/kernel_bench.py --only sketch --reps 1 > gpurun_out/ncu_sk1.log 2>&1
echo done
