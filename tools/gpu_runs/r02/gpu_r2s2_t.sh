# run T: decode cluster sizing with the light config (FP8Q_SKINNY_CLQ=1) vs default
timeout 300 python tools/kernel_bench.py --what none --decode --graph --flush read > gpurun_out/t_base.txt 2>&1
FP8Q_SKINNY_CLQ=1 FP8Q_DEBUG_CLUSTER=1 timeout 300 python tools/kernel_bench.py --what none --decode --graph --flush read > gpurun_out/t_clq.txt 2> gpurun_out/t_clq.err
FP8Q_SKINNY_CLQ=1 timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_linear.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/t_tests.txt
