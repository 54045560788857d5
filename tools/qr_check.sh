# QRCP check: parity tests (cluster tail on and off) + timings (+ trace)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_golden.py tests/test_gpu_cqrrpt.py -x -q -m gpu 2>&1 | tail -3
CQRRPT_QRCP_NOCLUSTER=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_golden.py -x -q -m gpu -k "qrcp or golden" 2>&1 | tail -2
for cfg in "131072 1024" "262144 2048" "16384 256" "4194304 256"; do
  set -- $cfg
  timeout 120 python tools/kernel_bench.py --only qrcp --m $1 --n $2
  CQRRPT_QRCP_NOCLUSTER=1 timeout 120 python tools/kernel_bench.py --only qrcp --m $1 --n $2
done
