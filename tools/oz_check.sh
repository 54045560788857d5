#!/bin/bash
# INT8 TRSM engine: its parity tests, then device time against the DMMA engine on the sizes quoted in DESIGN.md.
mkdir -p gpurun_out; out=gpurun_out/oz_check.log; : > $out
timeout 900 python -m pytest tests/test_gpu_oztrsm.py -q -m gpu --timeout 600 -x > gpurun_out/oz_check_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/oz_check_pytest.log
for sv in ${STAGES:-48 38 66}; do CQRRPT_OZ_STAGES=$sv python tools/oz_time.py 1048576 2048 >> $out 2>&1; done
timeout 600 python tools/oz_probe.py 262144 1024 1048576 2048 2097152 1024 1048576 512 524288 768 >> $out 2>&1
