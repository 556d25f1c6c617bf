# A/B: fused decode prologue with its activation loads batched 4 groups per warp (new) vs HEAD (base)
timeout 900 python -m pytest tests -m gpu -q -x -k "linear" 2>&1 | tail -4 > gpurun_out/s3_batch_tests.txt
for rep in 1 2; do
  for lib in base new; do
    if [ $lib = base ]; then export FP8Q_LIB=$PWD/paper_2601_18150_b200/libfp8q_base.so; else unset FP8Q_LIB; fi
    timeout 300 python bench.py --workload decode > gpurun_out/s3_batch_${lib}_${rep}.json 2> gpurun_out/s3_batch_${lib}_${rep}.err
  done
done
