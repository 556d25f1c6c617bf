mkdir -p gpurun_out
FP8Q_GEMV=1 timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q -k "skinny or decode" > gpurun_out/gemv2_parity.log 2>&1; echo parity=$?; tail -2 gpurun_out/gemv2_parity.log
echo "== gemv"; FP8Q_GEMV=1 timeout 600 python tools/kernel_bench.py --what none --decode --graph --flush read | grep -E '"shape": \[1,'
echo "== tensor"; timeout 600 python tools/kernel_bench.py --what none --decode --graph --flush read | grep -E '"shape": \[1,'
