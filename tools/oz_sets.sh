#!/bin/bash
# INT8 TRSM engine: one vs two drain sets (CQRRPT_OZ_SETS), correctness first.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_oztrsm.py -q -m gpu --timeout 600 -x > gpurun_out/oz_sets_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/oz_sets_pytest.log
for s in 1 2; do
  echo "sets=$s" >> gpurun_out/oz_sets.log
  CQRRPT_OZ_SETS=$s timeout 600 python tools/oz_probe.py 262144 1024 1048576 2048 2097152 1024 >> gpurun_out/oz_sets.log 2>&1
done
