# run Q: raster band sweep for the prefill GEMM (time per shape, cold L2) + down_proj DRAM traffic per band
for r in 0 4 6 8 12 16 24 32; do
  if [ $r = 0 ]; then unset FP8Q_GEMM_RASTER; else export FP8Q_GEMM_RASTER=$r; fi
  echo "raster=$r $(timeout 300 python tools/kernel_bench.py --what gemm --flush read 2>&1 | python -c 'import sys,json; print(" ".join(str(json.loads(l)["TFLOPs"]) for l in sys.stdin if l.startswith("{")))')" >> gpurun_out/q_raster.txt
done
unset FP8Q_GEMM_RASTER
for r in 0 4 8 16 32; do
  if [ $r = 0 ]; then unset FP8Q_GEMM_RASTER; else export FP8Q_GEMM_RASTER=$r; fi
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:pair_kernel --csv python tools/prof_kernels.py > gpurun_out/q_traffic_$r.csv 2>&1
done
