# dev sweep: decode weight stages prefetched before griddepcontrol.wait, with the fused m <= 16 path
for rep in 1 2; do
  for pf in 2 4 6 8; do
    FP8Q_SKINNY_PREFETCH=$pf timeout 300 python bench.py --workload decode > gpurun_out/s3_pf2_${pf}_${rep}.json 2> /dev/null
  done
done
