mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q -k "not skinny and not grouped" > gpurun_out/gemm_parity.log 2>&1; echo parity=$?
tail -1 gpurun_out/gemm_parity.log
timeout 300 python tools/kernel_bench.py --what gemm --flush read 2>&1 | grep TFLOP
FP8Q_GEMM_DEBUG=1 timeout 120 python tools/gemm_trace.py 8192 24576 4096 2>&1 | tail -6
