# dev: decode M = 129..256 on the swap-AB cluster kernel -- parity + timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/gemm_parity.log 2>&1; echo parity=$?
tail -2 gpurun_out/gemm_parity.log
echo "== trace 256 4096 4096"; timeout 120 python tools/skinny_trace.py 256 4096 4096 2>&1 | head -4
echo "== decode"; timeout 600 python tools/kernel_bench.py --what none --decode --graph --flush read | grep '"shape": \[256'
