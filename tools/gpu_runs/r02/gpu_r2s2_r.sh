# run R: KV cache kernels with one row per warp (grid up to 8 CTAs/SM): parity + timing A/B vs base
timeout 900 python -m pytest tests/test_gpu_kv.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r_kvtests.txt
FP8Q_LIB=$PWD/ab/libfp8q_base.so timeout 300 python tools/kernel_bench.py --what kv --flush read > gpurun_out/r_kv_base.txt 2>&1
timeout 300 python tools/kernel_bench.py --what kv --flush read > gpurun_out/r_kv_new.txt 2>&1
