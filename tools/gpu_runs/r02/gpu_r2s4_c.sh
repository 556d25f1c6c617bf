# session 4: tail split A/B -- current build (split on / off) vs the HEAD build, graph timings
S="256,24576,4096 128,24576,4096 64,24576,4096 8192,768,4096 8192,256,4096 8192,6144,4096 8192,640,2048 2048,512,4096"
python paper_2601_18150_b200/build.py > gpurun_out/s4c_build.txt 2>&1
timeout 300 python tools/one_shape.py $S > gpurun_out/s4c_cur.txt 2>&1
FP8Q_TAIL_SPLIT=0 timeout 300 python tools/one_shape.py $S > gpurun_out/s4c_cur_nosplit.txt 2>&1
FP8Q_LIB=$PWD/paper_2601_18150_b200/libfp8q_head.so timeout 300 python tools/one_shape.py $S > gpurun_out/s4c_head.txt 2>&1
timeout 300 python tools/one_shape.py $S > gpurun_out/s4c_cur2.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_shards.py tests/test_gpu_linear.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -5 > gpurun_out/s4c_tests.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/s4c_launches.csv python tools/one_shape.py 256,24576,4096 > /dev/null 2>&1
