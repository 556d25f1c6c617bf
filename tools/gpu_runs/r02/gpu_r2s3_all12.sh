# A/B: decode cluster reduction by all 12 warps (new) vs the 8 promotion warps (base)
timeout 900 python -m pytest tests -m gpu -q -x -k "linear or skinny or decode or gemm" 2>&1 | tail -4 > gpurun_out/s3_all12_tests.txt
for rep in 1 2; do
  for lib in base new; do
    if [ $lib = base ]; then export FP8Q_LIB=$PWD/paper_2601_18150_b200/libfp8q_base.so; else unset FP8Q_LIB; fi
    timeout 300 python bench.py --workload decode > gpurun_out/s3_all12_${lib}_${rep}.json 2> gpurun_out/s3_all12_${lib}_${rep}.err
  done
done
