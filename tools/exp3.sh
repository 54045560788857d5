#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_oztrsm.py -q -m gpu --timeout 600 -x > gpurun_out/exp3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/exp3_pytest.log
timeout 600 python tools/oz_probe.py 1000 300 70001 513 262144 1024 1048576 2048 2097152 1024 1048576 512 > gpurun_out/oz_n16.log 2>&1
