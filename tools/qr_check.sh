# QRCP check: parity tests (cluster tail on and off) + timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_golden.py tests/test_gpu_cqrrpt.py -x -q -m gpu 2>&1 | tail -3
CQRRPT_QRCP_NOCLUSTER=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_golden.py -x -q -m gpu -k "qrcp or golden" 2>&1 | tail -2
for cfg in "131072 1024" "262144 2048" "16384 256" "1048576 4096"; do
  set -- $cfg
  timeout 300 python tools/kernel_bench.py --only qrcp --m $1 --n $2
done
