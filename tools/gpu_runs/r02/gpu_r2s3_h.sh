# run 3H: B-resident raster (n-tile bands) for B < A GEMMs (down/qkv/o) vs the m-band raster -- tests, isolated GEMMs, step, DRAM bytes
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_shards.py tests/test_gpu_bench_e2e.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/h3_tests.txt
for b in 1 0; do
  FP8Q_GEMM_BRES=$b timeout 300 python tools/kernel_bench.py --what gemm > gpurun_out/h3_kgemm_$b.txt 2>&1
done
for b in 1 0 1 0; do
  FP8Q_GEMM_BRES=$b timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-e2e --no-cpu-baseline >> gpurun_out/h3_step_$b.json 2>> gpurun_out/h3_step.err
done
for b in 1 0; do
  FP8Q_GEMM_BRES=$b timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/h3_launches_$b.csv python bench.py --steps 2 --warmup 1 --no-extras --no-e2e --no-cpu-baseline > gpurun_out/h3_ncu_$b.log 2>&1
done
