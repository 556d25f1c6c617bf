# run C: NEXT-2 exact producers -- parity and timing
timeout 900 python -m pytest tests/test_gpu_producers.py -m gpu -q -x 2>&1 | tail -25 > gpurun_out/c_prod.txt
timeout 300 python tools/prod_bench.py > gpurun_out/c_prodbench.txt 2>&1
