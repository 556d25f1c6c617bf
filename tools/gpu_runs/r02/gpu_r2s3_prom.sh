# A/B: GEMM promotion with eight 16-column chunks through four slots (buffer handed back after 64 of 128 FMAs) (new) vs HEAD (base)
timeout 1200 python -m pytest tests -m gpu -q -x -k "gemm or linear or shard or e2e or fullsize or grouped or moe" 2>&1 | tail -3 > gpurun_out/s3_pr_tests.txt
for rep in 1 2 3; do
  for lib in base new; do
    if [ $lib = base ]; then export FP8Q_LIB=$PWD/paper_2601_18150_b200/libfp8q_base.so; else unset FP8Q_LIB; fi
    timeout 300 python bench.py --steps 20 --warmup 5 --no-extras --no-e2e --no-cpu-baseline > gpurun_out/s3_pr_${lib}_${rep}.json 2> gpurun_out/s3_pr_${lib}_${rep}.err
  done
done
for lib in base new; do
  if [ $lib = base ]; then export FP8Q_LIB=$PWD/paper_2601_18150_b200/libfp8q_base.so; else unset FP8Q_LIB; fi
  timeout 300 python tools/kernel_bench.py --what gemm --iters 20 > gpurun_out/s3_prk_${lib}.txt 2>&1
  timeout 300 python bench.py --workload moe > gpurun_out/s3_prm_${lib}.json 2>&1
done
