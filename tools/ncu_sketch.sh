#!/bin/bash
# sketch kernel: plain timings, then ncu captures (C2 exact, C5-256 split)
set -u
python tools/kernel_bench.py --only sketch > gpurun_out/kb_sketch.log 2>&1 || exit 1
python tools/kernel_bench.py --only sketch --m 4194304 --n 256 --fast-sketch >> gpurun_out/kb_sketch.log 2>&1 || exit 1
NCU="ncu --set full --clock-control none --import-source on -k regex:saso_apply -s 1 -c 1"
$NCU -o gpurun_out/prof_sketch_c2 python tools/kernel_bench.py --only sketch --reps 1 > gpurun_out/ncu_sk1.log 2>&1
$NCU -o gpurun_out/prof_sketch_c5 python tools/kernel_bench.py --only sketch --reps 1 --m 4194304 --n 256 --fast-sketch > gpurun_out/ncu_sk2.log 2>&1
echo done
