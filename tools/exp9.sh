#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/exp9.log; : > $out
timeout 900 python -m pytest tests/test_gpu_oztrsm.py -q -m gpu --timeout 600 -x > gpurun_out/exp9_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/exp9_pytest.log
for sv in 38 47 56; do CQRRPT_OZ_STAGES=$sv python tools/oz_time.py 1048576 2048 >> $out 2>&1; done
CQRRPT_OZ_DBG=1 python tools/oz_time.py 1048576 2048 >> $out 2>&1
timeout 600 python tools/oz_probe.py 262144 1024 1048576 2048 >> $out 2>&1
