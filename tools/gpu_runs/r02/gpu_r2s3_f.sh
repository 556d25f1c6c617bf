# run 3F: decode layer A/B -- trigger (entry / late) x ring (light, 2 CTAs per SM / full, 1 per SM), ordered stream-K
for cfg in "e_l::1" "late_l:late:1" "e_f::0" "late_f:late:0" "e_l2::1" "late_l2:late:1" "e_f2::0" "late_f2:late:0"; do
  IFS=: read name trig light <<< "$cfg"
  FP8Q_SKINNY_TRIGGER=$trig FP8Q_SKINNY_LIGHT=$light timeout 600 python bench.py --workload decode > gpurun_out/f3_$name.json 2> gpurun_out/f3_$name.err
done
FP8Q_TIMELINE_NPZ=gpurun_out/f3_late_f.npz FP8Q_SKINNY_TRIGGER=late FP8Q_SKINNY_LIGHT=0 timeout 300 python tools/decode_timeline.py --m 1 > gpurun_out/f3_tl_late_f.txt 2>&1
