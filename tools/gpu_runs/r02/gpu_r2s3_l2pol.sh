# A/B: L2 eviction policy of the quantizer / GEMM output streams (FP8Q_L2POL bitmask), headline step only
for rep in 1 2; do
  for pol in 0 1 3 5 7; do
    FP8Q_L2POL=$pol timeout 300 python bench.py --steps 20 --warmup 5 --no-extras --no-e2e --no-cpu-baseline > gpurun_out/s3_l2pol_${pol}_${rep}.json 2> gpurun_out/s3_l2pol_${pol}_${rep}.err
  done
done
