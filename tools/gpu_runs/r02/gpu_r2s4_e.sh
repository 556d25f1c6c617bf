# session 4: tail split with bulk-copy fixup through the idle ring -- A/B split on / off, then GEMM tests
S="256,24576,4096 128,24576,4096 64,24576,4096 8192,768,4096 8192,256,4096 8192,6144,4096 8192,640,2048 2048,512,4096 200,24576,2048"
python paper_2601_18150_b200/build.py > gpurun_out/s4e_build.txt 2>&1
timeout 300 python tools/one_shape.py $S > gpurun_out/s4e_cur.txt 2>&1
FP8Q_TAIL_SPLIT=0 timeout 300 python tools/one_shape.py $S > gpurun_out/s4e_nosplit.txt 2>&1
timeout 300 python tools/one_shape.py $S > gpurun_out/s4e_cur2.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_shards.py -q -x 2>&1 | tail -5 > gpurun_out/s4e_tests.txt
