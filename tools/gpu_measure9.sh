# dev: decode cluster mode with the full-budget config at M <= 32 (A/B vs light)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q -k "skinny or decode" > gpurun_out/gemm_parity.log 2>&1; echo parity=$?
tail -2 gpurun_out/gemm_parity.log
echo "== heavy"; timeout 600 python tools/kernel_bench.py --what none --decode --graph --flush read | grep -E '"shape": \[(1|8),'
echo "== light"; FP8Q_SKINNY_LIGHT_CLUSTER=1 timeout 600 python tools/kernel_bench.py --what none --decode --graph --flush read | grep -E '"shape": \[(1|8),'
