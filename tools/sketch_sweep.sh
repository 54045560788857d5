#!/bin/bash
# SASO apply variants: row-block width A and staging path, per config.
for cfg in C2 C3 C4 C5_256 C5_1024 C5_2048; do
  for A in default 12 16; do
    for path in LDGSTS TMA; do
      envs=""
      [ "$A" != "default" ] && envs="CQRRPT_SASO_A=$A"
      [ "$path" = "LDGSTS" ] && envs="$envs CQRRPT_SASO_LDGSTS=1" || envs="$envs CQRRPT_SASO_TMA=1"
      echo -n "$cfg A=$A $path: "
      env $envs python tools/sketch_bench.py $cfg 2>&1 | tail -1
    done
  done
done
