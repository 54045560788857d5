#!/bin/bash
# SASO apply at the wide configs: forced column-group width W and A vs the default choice.
mkdir -p gpurun_out
out=gpurun_out/sketch_w2.log; : > $out
run() { echo "== $*" >> $out; env "${@:4}" python tools/sketch_bench.py $1,$2,$3 >> $out 2>&1; }
for shape in "4194304 2048 2560" "1048576 4096 5120" "4194304 1024 1280" "262144 2048 2560" "131072 1024 1280"; do
  run $shape X=0
  for w in 16 8; do for a in 8 12 16; do run $shape CQRRPT_SASO_W=$w CQRRPT_SASO_A=$a; done; done
done
