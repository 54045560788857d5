#!/bin/bash
# Round-2 end evidence: smoke + whole -m gpu suite + default bench + reference
# arm (tools/final_check.sh), every secondary config's bench line, the ncu
# launch list / DRAM traffic of the default config, one ncu --set full of the
# INT8 update kernel at m = 1M, k = 2048.
mkdir -p gpurun_out
bash tools/final_check.sh
for cfg in C1 C2 C3 C3b C4 C5_256 C5_512 C5_1024; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
done
bash tools/ncu_bench.sh C5_2048
CQRRPT_GPU_TRSM=oz timeout 900 ncu --set full --clock-control none --import-source on -k regex:oz_update -s 8 -c 1 \
    -o gpurun_out/oz_update_final python tools/oz_one.py 1048576 2048 > gpurun_out/ncu_oz_final.log 2>&1
echo done
