# session 4: decode M = 129..256 on the CTA pair with the tail split (variant build: M >= 256 plan gate, no swap-AB above M = 128) vs default
S="256,4096,12288 256,4096,4096 256,6144,4096 256,24576,4096 200,4096,12288 160,6144,4096"
V=$PWD/paper_2601_18150_b200/libfp8q_m256.so
timeout 300 python tools/one_shape.py $S > gpurun_out/s4m_def.txt 2>&1
FP8Q_LIB=$V timeout 300 python tools/one_shape.py $S > gpurun_out/s4m_var.txt 2>&1
timeout 300 python tools/one_shape.py $S > gpurun_out/s4m_def2.txt 2>&1
FP8Q_LIB=$V timeout 300 python tools/one_shape.py $S > gpurun_out/s4m_var2.txt 2>&1
