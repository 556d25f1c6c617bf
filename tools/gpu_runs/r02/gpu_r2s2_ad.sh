# run AD: MoE next-tile L2 prefetch (one-CTA grouped kernel) -- grouped parity + MoE timing A/B vs base
timeout 1200 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_fullsize.py -m gpu -q -x -k "group or moe or grouped or qwen3_30b" 2>&1 | tail -3 > gpurun_out/ad_tests.txt
FP8Q_LIB=$PWD/ab/libfp8q_base.so timeout 300 python tools/kernel_bench.py --what none --moe --flush read > gpurun_out/ad_moe_base.txt 2>&1
timeout 300 python tools/kernel_bench.py --what none --moe --flush read > gpurun_out/ad_moe_new.txt 2>&1
