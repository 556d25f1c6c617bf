# run AE: act quantizer per-item overhead cut (producer metadata, 32-bit indices, predicated stores,
# warp-uniform fast path) -- exhaustive + parity, timing A/B vs base, in-step bench
timeout 1500 python -m pytest tests/test_gpu_exhaustive.py tests/test_gpu_quant.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/ae_tests.txt
for i in 1 2; do
FP8Q_LIB=$PWD/ab/libfp8q_base.so timeout 300 python tools/kernel_bench.py --what aq --flush read > gpurun_out/ae_aq_base_$i.txt 2>&1
timeout 300 python tools/kernel_bench.py --what aq --flush read > gpurun_out/ae_aq_new_$i.txt 2>&1
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/ae_bench.json 2> gpurun_out/ae_bench.err
FP8Q_LIB=$PWD/ab/libfp8q_base.so timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/ae_bench_base.json 2> gpurun_out/ae_bench_base.err
