# run S: chunked / reordered e2e pipeline -- parity vs the device step, then the bench line
timeout 900 python -m pytest tests/test_gpu_bench_e2e.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/s_tests.txt
timeout 900 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err
