#!/bin/bash
# Round-2 evidence: new engine tests, default bench line, secondary configs,
# ncu launch list + DRAM traffic of the default config.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_oztrsm.py -q -m gpu > gpurun_out/oz_tests.log 2>&1; echo "rc=$?" >> gpurun_out/oz_tests.log
timeout 900 python bench.py > gpurun_out/bench_c5_2048.json 2> gpurun_out/bench_c5_2048.err
for cfg in C1 C2 C3 C4 C5_256 C5_512 C5_1024; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
done
if [ "${NCU:-1}" = 1 ]; then bash tools/ncu_bench.sh C5_2048; fi
