# session 4: CTA-pair tail-wave split (plan_pair_split) -- parity, then A/B vs FP8Q_PAIR_SPLIT=0
python paper_2601_18150_b200/build.py > gpurun_out/s4b_build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_shards.py -q -x 2>&1 | tail -15 > gpurun_out/s4b_tests.txt
timeout 600 python tools/kernel_bench.py --what none --decode --graph --iters 10 > gpurun_out/s4b_dec_split.txt 2>&1
FP8Q_PAIR_SPLIT=0 timeout 600 python tools/kernel_bench.py --what none --decode --graph --iters 10 > gpurun_out/s4b_dec_nosplit.txt 2>&1
timeout 600 python tools/shard_bench.py > gpurun_out/s4b_shard_split.txt 2>&1
FP8Q_PAIR_SPLIT=0 timeout 600 python tools/shard_bench.py > gpurun_out/s4b_shard_nosplit.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/s4b_bench_split.json 2>/dev/null
FP8Q_PAIR_SPLIT=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/s4b_bench_nosplit.json 2>/dev/null
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/s4b_bench_split2.json 2>/dev/null
