# A/B at the unthrottled clock: whole-model sync (sync8b / sync30b) and isolated weight quantization,
# staged weight kernel of 2cce46d (base) vs HEAD (new)
for rep in 1 2; do
  for lib in base new; do
    if [ $lib = base ]; then export FP8Q_LIB=$PWD/paper_2601_18150_b200/libfp8q_base.so; else unset FP8Q_LIB; fi
    timeout 300 python bench.py --workload sync8b > gpurun_out/s3_wq2_8b_${lib}_${rep}.json 2>&1
    timeout 300 python bench.py --workload sync30b > gpurun_out/s3_wq2_30b_${lib}_${rep}.json 2>&1
  done
done
