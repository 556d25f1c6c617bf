# A/B: decode cluster split-K reduction -- RU units' DSMEM loads per peer in flight, 8/16-byte output stores (new) vs HEAD (base)
timeout 1200 python -m pytest tests -m gpu -q -x -k "gemm or linear or skinny or decode or shard" 2>&1 | tail -3 > gpurun_out/s3_dsm_tests.txt
for rep in 1 2; do
  for lib in base new; do
    if [ $lib = base ]; then export FP8Q_LIB=$PWD/paper_2601_18150_b200/libfp8q_base.so; else unset FP8Q_LIB; fi
    timeout 300 python bench.py --workload decode > gpurun_out/s3_dsm_${lib}_${rep}.json 2> gpurun_out/s3_dsm_${lib}_${rep}.err
  done
done
