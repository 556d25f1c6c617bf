# session 4: tail split (pair, M >= 1024, >= 8 k-blocks per slice) -- GPU suite, A/B, bench line
S="8192,768,4096 8192,256,4096 8192,6144,4096 8192,640,2048 2048,512,4096 8192,512,4096 8192,1280,2048 8192,1536,4096"
python paper_2601_18150_b200/build.py > gpurun_out/s4f_build.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/s4f_gputests.txt
timeout 300 python tools/one_shape.py $S > gpurun_out/s4f_cur.txt 2>&1
FP8Q_TAIL_SPLIT=0 timeout 300 python tools/one_shape.py $S > gpurun_out/s4f_nosplit.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s4f_bench.json 2> gpurun_out/s4f_bench.err
FP8Q_TAIL_SPLIT=0 timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s4f_bench_nosplit.json 2> /dev/null
