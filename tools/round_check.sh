#!/bin/bash
# Full GPU check: smoke, all gpu tests, bench (1 GPU), phase timings, launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -x -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python tools/phase_timing.py ${PHASES:-C1 C2} > gpurun_out/phases.jsonl 2> gpurun_out/phases.err; echo "phases rc=$?" >> gpurun_out/phases.err
if [ -n "${QRCP_TRACE:-}" ]; then
  CQRRPT_QRCP_TRACE=1 timeout 300 python tools/phase_timing.py $QRCP_TRACE --reps 1 > /dev/null 2> gpurun_out/qrcp_trace.log
fi
if [ "${NCU_LIST:-1}" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_list.log
fi
