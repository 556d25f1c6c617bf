mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/gemm_parity.log 2>&1; echo parity=$?
tail -1 gpurun_out/gemm_parity.log
timeout 300 python tools/kernel_bench.py --what gemm --flush read 2>&1 | grep TFLOP
FP8Q_GEMM_DEBUG=1 timeout 300 python tools/kernel_bench.py --what gemm --flush read 2>&1 | grep 24576
timeout 300 python tools/kernel_bench.py --what none --moe --flush read 2>&1 | grep '"T": 8192, "skew": 0.0'
timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('layer', d['value'], d['breakdown'])"
