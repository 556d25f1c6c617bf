# A/B: B loads with an L2 evict_last hint under the B-resident raster (FP8Q_GEMM_BLAST=1) -- DRAM bytes per GEMM launch and step time
for v in 0 1; do
  FP8Q_GEMM_BLAST=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/s3_blast_l$v.csv python bench.py --steps 2 --warmup 1 --no-extras --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
for rep in 1 2; do
  for v in 0 1; do
    FP8Q_GEMM_BLAST=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-extras --no-e2e --no-cpu-baseline > gpurun_out/s3_blast_${v}_${rep}.json 2> /dev/null
  done
done
FP8Q_GEMM_BLAST=1 timeout 900 python -m pytest tests -m gpu -q -x -k "gemm" 2>&1 | tail -2 > gpurun_out/s3_blast_tests.txt
