mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/gemv_parity.log 2>&1; echo parity=$?; tail -3 gpurun_out/gemv_parity.log
echo "== gemv"; timeout 600 python tools/kernel_bench.py --what none --decode --graph --flush read | grep -E '"shape": \[1,'
echo "== tensor"; FP8Q_GEMV=0 timeout 600 python tools/kernel_bench.py --what none --decode --graph --flush read | grep -E '"shape": \[1,'
