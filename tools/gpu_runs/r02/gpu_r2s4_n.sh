# session 4: decode M = 256 qkv / down on the split CTA pair (dispatch) -- GPU suite, decode A/B
python paper_2601_18150_b200/build.py > gpurun_out/s4n_build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/s4n_gputests.txt
S="256,4096,12288 256,4096,4096 256,6144,4096 256,24576,4096 512,4096,4096"
timeout 300 python tools/one_shape.py $S > gpurun_out/s4n_cur.txt 2>&1
FP8Q_TAIL_SPLIT=0 timeout 300 python tools/one_shape.py $S > gpurun_out/s4n_nosplit.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s4n_bench.json 2> gpurun_out/s4n_bench.err
FP8Q_TAIL_SPLIT=0 timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s4n_bench_nosplit.json 2> /dev/null
