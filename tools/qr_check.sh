# QRCP check: parity tests + timings (+ trace)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_golden.py tests/test_gpu_cqrrpt.py -x -q -m gpu 2>&1 | tail -3
timeout 120 python tools/kernel_bench.py --only qrcp
timeout 120 python tools/kernel_bench.py --only qrcp --m 262144 --n 2048
timeout 120 python tools/kernel_bench.py --only qrcp --m 16384 --n 256
CQRRPT_QRCP_TRACE=1 timeout 300 python tools/phase_timing.py C2 --reps 1 > /dev/null 2> gpurun_out/qrcp_trace.log
