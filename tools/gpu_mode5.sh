for d in 0 1 5 3; do
echo "== debug $d"; FP8Q_GEMM_DEBUG=$d timeout 300 python tools/kernel_bench.py --what gemm --flush read 2>&1 | grep -E '24576|12288\]'
done
