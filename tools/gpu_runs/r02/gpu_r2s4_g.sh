# session 4: tail split (pair, M >= 1024, >= 16 k-blocks per slice) -- GPU suite, bench A/B x2
python paper_2601_18150_b200/build.py > gpurun_out/s4g_build.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/s4g_gputests.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s4g_bench.json 2> gpurun_out/s4g_bench.err
FP8Q_TAIL_SPLIT=0 timeout 900 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/s4g_bench_nosplit.json 2> /dev/null
timeout 900 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/s4g_bench2.json 2> /dev/null
FP8Q_TAIL_SPLIT=0 timeout 900 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/s4g_bench_nosplit2.json 2> /dev/null
