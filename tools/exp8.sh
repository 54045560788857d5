#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
CQRRPT_GPU_TRSM=oz ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"oz_|trsm_block" python tools/oz_one.py 1048576 2048 > gpurun_out/oz_launches.csv 2>&1
CQRRPT_GPU_TRSM=oz timeout 900 ncu --set full --clock-control none --import-source on -k regex:oz_update -s 8 -c 1 -f \
    -o gpurun_out/oz_update_n16 python tools/oz_one.py 1048576 2048 > gpurun_out/ncu_oz_n16.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:saso_apply -s 1 -c 1 -f \
    -o gpurun_out/saso_c5_256 python tools/sketch_one.py 4194304 256 320 > gpurun_out/ncu_saso_c5_256.log 2>&1
