#!/bin/bash
# sketch kernel: plain timing, then one ncu --set full capture (C2 shape)
python tools/kernel_bench.py --only sketch > gpurun_out/kb_sketch.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"saso_apply" -s 1 -c 1 -o gpurun_out/prof_sketch2 \
  python tools/kernel_bench.py --only sketch --reps 1 > gpurun_out/ncu_sketch2.log 2>&1
echo done
