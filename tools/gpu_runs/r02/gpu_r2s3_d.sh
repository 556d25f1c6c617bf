# run 3D: decode timeline with SM placement (ordered stream-K), default and late trigger
timeout 300 python tools/decode_timeline.py --m 1 > gpurun_out/d3_tl_m1.txt 2>&1
FP8Q_SKINNY_TRIGGER=late timeout 300 python tools/decode_timeline.py --m 1 > gpurun_out/d3_tl_m1_late.txt 2>&1
timeout 300 python tools/decode_timeline.py --m 64 > gpurun_out/d3_tl_m64.txt 2>&1
