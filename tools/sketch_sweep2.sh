#!/bin/bash
# SASO apply: row-block width A x staging path on the narrow / large-d shapes,
# then ncu counters of the default choice.
mkdir -p gpurun_out
for cfg in C5_256 C4 C2; do
  for A in 1 2 4 8 16; do
    for path in LDGSTS TMA; do
      envs="CQRRPT_SASO_A=$A"
      [ "$path" = "LDGSTS" ] && envs="$envs CQRRPT_SASO_LDGSTS=1" || envs="$envs CQRRPT_SASO_TMA=1"
      echo -n "$cfg A=$A $path: "
      env $envs timeout 120 python tools/sketch_bench.py $cfg 2>&1 | tail -1
    done
  done
done
M="gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size"
for shape in "4194304 256 320" "1048576 4096 5120" "131072 1024 1280"; do
  echo "ncu $shape"
  timeout 300 ncu --metrics $M --clock-control none --csv -k regex:saso_apply python tools/sketch_one.py $shape 2>/dev/null | grep saso_apply | tail -7
done
