#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/exp10.log; : > $out
for g in dmma ozaki; do
  for cfg in C5_512 C5_256; do
    echo "== $cfg gram=$g" >> $out
    CQRRPT_GPU_GRAM=$g timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(j['ms_per_step'],2), j['phases_ms'])" >> $out 2>&1
  done
done
for t in dmma oz; do
  echo "== C5_512 trsm=$t" >> $out
  CQRRPT_GPU_TRSM=$t timeout 600 python bench.py --config C5_512 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(j['ms_per_step'],2), j['phases_ms'])" >> $out 2>&1
done
