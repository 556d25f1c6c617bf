# run AH: fractional-wave prefill shapes on the one-CTA kernel split along K -- parity + shard timing A/B
timeout 1200 python -m pytest tests/test_gpu_shards.py tests/test_gpu_gemm.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/ah_tests.txt
FP8Q_LIB=$PWD/ab/libfp8q_base.so timeout 300 python tools/shard_bench.py > gpurun_out/ah_sh_base.txt 2>&1
timeout 300 python tools/shard_bench.py > gpurun_out/ah_sh_new.txt 2>&1
