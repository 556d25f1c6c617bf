timeout 900 python -m pytest tests/test_gpu_bench_e2e.py -m gpu -q 2>&1 | grep -E "Error|passed|failed" | head -12 > gpurun_out/s3_tests.txt
