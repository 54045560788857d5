#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/exp5.log; : > $out
for d in 0 1 2 4 8 12 3 15; do CQRRPT_OZ_DBG=$d python tools/oz_time.py 1048576 2048 >> $out 2>&1; done
for sv in 28 38 46 55 64 82; do CQRRPT_OZ_STAGES=$sv python tools/oz_time.py 1048576 2048 >> $out 2>&1; done
for sv in 28 46 64 82; do CQRRPT_OZ_DBG=15 CQRRPT_OZ_STAGES=$sv python tools/oz_time.py 1048576 2048 >> $out 2>&1; done
CQRRPT_GPU_TRSM=dmma python tools/oz_time.py 1048576 2048 >> $out 2>&1
