# dev: decode cluster split-K -- parity, per-CTA timeline, graph timing A/B vs stream-K
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/gemm_parity.log 2>&1; echo parity=$?
tail -5 gpurun_out/gemm_parity.log
for mnk in "1 6144 4096" "64 6144 4096" "128 4096 4096"; do
echo "== trace $mnk"; timeout 120 python tools/skinny_trace.py $mnk 2>&1 | head -4
done
echo "== decode cluster"; timeout 600 python tools/kernel_bench.py --what none --decode --graph --flush read
echo "== decode streamk"; FP8Q_SKINNY_CLUSTER=0 timeout 600 python tools/kernel_bench.py --what none --decode --graph --flush read
