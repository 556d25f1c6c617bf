for d in 0 4 1; do
echo "== debug $d"; FP8Q_GEMM_DEBUG=$d timeout 300 python tools/kernel_bench.py --what gemm --flush read 2>&1 | grep 24576
FP8Q_GEMM_DEBUG=$d timeout 120 python tools/gemm_trace.py 8192 24576 4096 2>&1 | sed -n '13,15p' | awk '{print $1, $3, $4, $5, $7, $13, $14, $16}'
done
