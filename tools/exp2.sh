#!/bin/bash
# round-2 experiment batch: wide-N MMAs in the INT8 TRSM engine, narrow column groups in the sketch
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_oztrsm.py tests/test_gpu_kernels.py -q -m gpu --timeout 600 -x > gpurun_out/exp2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/exp2_pytest.log
: > gpurun_out/oz_sets.log
for s in 1 2; do
  echo "sets=$s" >> gpurun_out/oz_sets.log
  CQRRPT_OZ_SETS=$s timeout 600 python tools/oz_probe.py 262144 1024 1048576 2048 2097152 1024 1048576 512 >> gpurun_out/oz_sets.log 2>&1
done
timeout 1200 bash tools/sketch_w.sh
