# round 2 / session 2, run A: GPU suite, default bench, GEMM kind A/B (1256 vs 2256 split pair)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/a_gputests.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err
for k in 1256 2256; do
  FP8Q_GEMM_KIND=$k timeout 300 python tools/kernel_bench.py --what gemm --flush read > gpurun_out/a_kind_$k.txt 2>&1
done
FP8Q_GEMM_KIND=1256 timeout 300 python tools/kernel_bench.py --what gemm --flush read > gpurun_out/a_kind_1256b.txt 2>&1
