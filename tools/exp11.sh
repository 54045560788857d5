#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/exp11.log; : > $out
for sp in 0 1 2 3; do echo "spin=$sp" >> $out; CQRRPT_OZ_SPIN=$sp python tools/oz_time.py 1048576 2048 >> $out 2>&1; done
CQRRPT_OZ_SPIN=3 timeout 600 python -m pytest tests/test_gpu_oztrsm.py -q -m gpu --timeout 600 -x > gpurun_out/exp11_pytest.log 2>&1
