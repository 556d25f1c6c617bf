# run AB: PDL in the producer-fused quantizers -- parity + timing
timeout 1200 python -m pytest tests/test_gpu_producers.py tests/test_gpu_quant.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/ab_tests.txt
timeout 300 python tools/prod_bench.py > gpurun_out/ab_prod.txt 2>&1
