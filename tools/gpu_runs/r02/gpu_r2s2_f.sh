# run F: fused decode activation quantization (fp8_linear_dynamic) -- parity, then decode timing
timeout 1200 python -m pytest tests/test_gpu_linear.py tests/test_gpu_gemm.py -m gpu -q -x 2>&1 | tail -20 > gpurun_out/f_tests.txt
timeout 600 python bench.py --workload decode > gpurun_out/f_decode.json 2> gpurun_out/f_decode.err
timeout 300 python tools/kernel_bench.py --what none --decode --graph --flush read > gpurun_out/f_kdecode.txt 2>&1
