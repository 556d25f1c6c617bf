# dev: two MMA-issuing warps (FP8Q_GEMM_DUAL=1) -- parity, A/B timing, trace, bench
mkdir -p gpurun_out
FP8Q_GEMM_DUAL=1 timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/gemm_dual_parity.log 2>&1; echo parity=$?
tail -2 gpurun_out/gemm_dual_parity.log
echo "== single"; timeout 300 python tools/kernel_bench.py --what gemm --flush read 2>&1 | grep TFLOP
echo "== dual"; FP8Q_GEMM_DUAL=1 timeout 300 python tools/kernel_bench.py --what gemm --flush read 2>&1 | grep TFLOP
echo "== dual debug1"; FP8Q_GEMM_DUAL=1 FP8Q_GEMM_DEBUG=1 timeout 300 python tools/kernel_bench.py --what gemm --flush read 2>&1 | grep 24576
FP8Q_GEMM_DUAL=1 timeout 120 python tools/gemm_trace.py 8192 24576 4096 2>&1 | sed -n '1p;12,16p' | awk '{print $1, $2, $3, $4, $5, $7, $13, $14, $15, $16}'
FP8Q_GEMM_DUAL=1 timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dual layer', d['value'], d['breakdown'])"
