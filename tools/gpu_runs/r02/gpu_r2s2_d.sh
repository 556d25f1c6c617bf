# run D: exact producers (tiny-g fix), GEMM after dev-mode removal, headline bench
timeout 900 python -m pytest tests/test_gpu_producers.py tests/test_gpu_gemm.py -m gpu -q -x 2>&1 | tail -15 > gpurun_out/d_tests.txt
FP8Q_GEMM_KIND=1256 timeout 300 python tools/kernel_bench.py --what gemm --flush read > gpurun_out/d_gemm.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/d_bench.json 2> gpurun_out/d_bench.err
