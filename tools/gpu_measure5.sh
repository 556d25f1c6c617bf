# dev: decode fixup batching -- parity + per-CTA timeline + graph timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/gemm_parity.log 2>&1; echo parity=$?
tail -3 gpurun_out/gemm_parity.log
for mnk in "1 6144 4096" "64 6144 4096" "128 4096 4096"; do
echo "== trace $mnk"; timeout 120 python tools/skinny_trace.py $mnk 2>&1 | head -10
done
echo "== decode"; timeout 600 python tools/kernel_bench.py --what none --decode --graph --flush read
