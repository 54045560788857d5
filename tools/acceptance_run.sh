#!/bin/bash
# The reference's acceptance suite, check by check, on the GPU drop-in
# (oracle/_ref/acceptance_gpu) and on the unmodified CPU library
# (oracle/_ref/acceptance_ref). Output: gpurun_out/acceptance.txt
out=gpurun_out/acceptance.txt
mkdir -p gpurun_out
echo "# host: $(nproc) cores; $(nvidia-smi --query-gpu=name --format=csv,noheader 2>/dev/null | head -1)" > $out
for impl in gpu ref; do
  echo "## acceptance_$impl (one process per check)" >> $out
  for c in thm2.1 thm2.2 cor3.1 stability rank pivots-low pivots-high rrqr-inherit maxnorm pivot-equiv flops sketch-struct; do
    timeout 600 oracle/_ref/acceptance_$impl --only $c 2>&1 | grep -E "^\[" | grep -v runtime >> $out
  done
done
cat $out
