# run AA: fused decode path removed (fp8_linear_dynamic = PDL-chained quantizer + GEMM): parity + decode
timeout 1500 python -m pytest tests/test_gpu_linear.py tests/test_gpu_gemm.py tests/test_gpu_quant.py tests/test_gpu_producers.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/aa_tests.txt
timeout 600 python bench.py --workload decode > gpurun_out/aa_decode.json 2> gpurun_out/aa_decode.err
