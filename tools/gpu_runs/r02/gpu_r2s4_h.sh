# session 4: tail split at M = 256 (variant build with the M >= 256 gate, FP8Q_LIB) vs the default build
S="256,24576,4096 512,24576,4096 256,12288,4096 768,6144,4096"
V=$PWD/paper_2601_18150_b200/libfp8q_m256.so
timeout 300 python tools/one_shape.py $S > gpurun_out/s4h_def.txt 2>&1
FP8Q_LIB=$V timeout 300 python tools/one_shape.py $S > gpurun_out/s4h_m256.txt 2>&1
timeout 300 python tools/one_shape.py $S > gpurun_out/s4h_def2.txt 2>&1
FP8Q_LIB=$V timeout 300 python tools/one_shape.py $S > gpurun_out/s4h_m256_2.txt 2>&1
