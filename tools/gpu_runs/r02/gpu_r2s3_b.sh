# run 3B: decode layer timeline from the trace build (libfp8q_trace.so), M = 1 / 64 / 128, and M = 1 with the late trigger
for m in 1 64 128; do timeout 300 python tools/decode_timeline.py --m $m > gpurun_out/b3_tl_m$m.txt 2>&1; done
FP8Q_SKINNY_TRIGGER=late timeout 300 python tools/decode_timeline.py --m 1 > gpurun_out/b3_tl_m1_late.txt 2>&1
