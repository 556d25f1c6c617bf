# dev: prefill GEMM tile kinds A/B (pair 256x256 = 1256, pair 256x128 = 1128 with 4 TMEM buffers)
timeout 600 env FP8Q_GEMM_KIND=1128 python -m pytest tests/test_gpu_gemm.py -x -q -k "not skinny and not grouped and not decode and not splitk" > gpurun_out/kind1128_parity.log 2>&1; echo parity1128=$?
tail -2 gpurun_out/kind1128_parity.log
for kind in 1256 1128; do
echo "== kind $kind"
FP8Q_GEMM_KIND=$kind timeout 300 python tools/kernel_bench.py --what gemm --flush read 2>&1 | grep TFLOP
done
echo "== trace 1128"
FP8Q_GEMM_KIND=1128 timeout 120 python tools/gemm_trace.py 8192 24576 4096 2>&1 | sed -n '1p;12,20p' | awk '{print $1, $2, $3, $4, $5, $7, $13, $14, $15, $16}'
