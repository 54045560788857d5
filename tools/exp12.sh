#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/exp12.log; : > $out
timeout 600 python -m pytest tests/test_gpu_oztrsm.py -q -m gpu --timeout 600 -x > gpurun_out/exp12_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/exp12_pytest.log
for sv in 48 38; do CQRRPT_OZ_STAGES=$sv python tools/oz_time.py 1048576 2048 >> $out 2>&1; done
timeout 600 python tools/oz_probe.py 262144 1024 1048576 2048 >> $out 2>&1
