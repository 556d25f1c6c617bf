# dev A/B: decode GEMM weight stages prefetched before griddepcontrol.wait (FP8Q_SKINNY_PREFETCH), decode layer record
for rep in 1 2; do
  for pf in all 0 2 4 6; do
    if [ $pf = all ]; then unset FP8Q_SKINNY_PREFETCH; else export FP8Q_SKINNY_PREFETCH=$pf; fi
    timeout 300 python bench.py --workload decode > gpurun_out/s3_pf_${pf}_${rep}.json 2> /dev/null
  done
done
