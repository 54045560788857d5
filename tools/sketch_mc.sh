#!/bin/bash
# SASO apply with / without multicast clusters, per config.
for cfg in C2 C3 C5_256 C5_1024 C4 C5_2048; do
  for v in "CQRRPT_SASO_MC=1" "X=1" "CQRRPT_SASO_MCTMA=1"; do
    echo -n "$cfg $v: "; env $v timeout 120 python tools/sketch_bench.py $cfg 2>&1 | tail -1
  done
done
