mkdir -p gpurun_out
for cfg in C5_2048 C4; do
  for eng in oz dmma; do
    CQRRPT_GPU_TRSM=$eng timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_${cfg}_${eng}.json 2> gpurun_out/b_${cfg}_${eng}.err
  done
done
CQRRPT_GPU_TRSM=oz timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -x > gpurun_out/pytest_oz.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_oz.log
