# run L: branch-free scale loads in the promotion loop -- GEMM parity + timing + headline
timeout 1200 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -4 > gpurun_out/l_tests.txt
FP8Q_GEMM_KIND=1256 timeout 300 python tools/kernel_bench.py --what gemm --flush read > gpurun_out/l_gemm.txt 2>&1
timeout 300 python tools/kernel_bench.py --what none --moe --flush read > gpurun_out/l_moe.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/l_bench.json 2> gpurun_out/l_bench.err
