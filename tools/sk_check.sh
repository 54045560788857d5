# sketch kernel check: parity tests + timings of both entry-loop variants
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_golden.py -x -q -m gpu -k "saso or sketch" 2>&1 | tail -2
CQRRPT_SASO_PIPE=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "saso or sketch" 2>&1 | tail -2
for P in "" 1; do
  if [ -n "$P" ]; then export CQRRPT_SASO_PIPE=1; else unset CQRRPT_SASO_PIPE; fi
  echo "PIPE=$P"
  timeout 120 python tools/kernel_bench.py --only sketch
  timeout 120 python tools/kernel_bench.py --only sketch --m 4194304 --n 256
  timeout 120 python tools/kernel_bench.py --only sketch --m 262144 --n 2048
done
