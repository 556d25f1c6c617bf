# dev: GEMM chain decomposition -- trace + TFLOP/s per debug mode (0 real, 1 no promotion,
# 2 no promotion + no TMA, 3 TMA + MMA without the release chain)
for d in 0 1 2 3; do
echo "== debug $d"
FP8Q_GEMM_DEBUG=$d timeout 120 python tools/gemm_trace.py 8192 24576 4096 2>&1 | sed -n '1p;12,16p' | awk '{print $1, $2, $3, $4, $5, $7, $13, $14, $15, $16}'
FP8Q_GEMM_DEBUG=$d timeout 300 python tools/kernel_bench.py --what gemm --flush read 2>&1 | grep 24576
done
