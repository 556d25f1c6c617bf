# run 3G: decode kernel with one CTA per SM, late dependent trigger, ordered stream-K -- GPU tests + decode layer x2 + timeline
timeout 1200 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_linear.py tests/test_gpu_shards.py tests/test_gpu_bench_e2e.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/g3_tests.txt
timeout 600 python bench.py --workload decode > gpurun_out/g3_dec1.json 2> gpurun_out/g3_dec1.err
timeout 600 python bench.py --workload decode > gpurun_out/g3_dec2.json 2> gpurun_out/g3_dec2.err
FP8Q_TIMELINE_NPZ=gpurun_out/g3_m1.npz timeout 300 python tools/decode_timeline.py --m 1 > gpurun_out/g3_tl_m1.txt 2>&1
