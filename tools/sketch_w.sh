#!/bin/bash
# SASO apply at the narrow-n configs: forced column-group width W and A vs the default choice.
mkdir -p gpurun_out
out=gpurun_out/sketch_w.log; : > $out
run() { # m n d, env...
  echo "== $*" >> $out
  env "${@:4}" python tools/sketch_bench.py $1,$2,$3 >> $out 2>&1
}
for shape in "4194304 256 320" "4194304 512 640" "4194304 256 256" "4194304 256 512"; do
  run $shape X=0
  for w in 8 16 32; do for a in 1 2 4 8; do run $shape CQRRPT_SASO_W=$w CQRRPT_SASO_A=$a; done; done
done
