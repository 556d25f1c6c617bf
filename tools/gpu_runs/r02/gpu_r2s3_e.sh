# run 3E: raw decode timelines (npz) for offline straggler analysis, early and late trigger, M = 1
FP8Q_TIMELINE_NPZ=gpurun_out/e3_m1.npz timeout 300 python tools/decode_timeline.py --m 1 > gpurun_out/e3_tl_m1.txt 2>&1
FP8Q_TIMELINE_NPZ=gpurun_out/e3_m1_late.npz FP8Q_SKINNY_TRIGGER=late timeout 300 python tools/decode_timeline.py --m 1 > gpurun_out/e3_tl_m1_late.txt 2>&1
nvidia-smi -q | grep -i -A3 "gpc\|MIG" | head -20 > gpurun_out/e3_smi.txt
