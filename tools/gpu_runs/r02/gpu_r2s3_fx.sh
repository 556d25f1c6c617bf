# fused activation quantization in the decode GEMM (fp8_linear_dynamic, m <= 16): parity + decode layer A/B (FP8Q_LINEAR_FUSED=0 = two launches)
timeout 900 python -m pytest tests -m gpu -q -x -k "linear or skinny or decode" 2>&1 | tail -15 > gpurun_out/s3_fx_tests.txt
for rep in 1 2; do
  for v in 0 1; do
    FP8Q_LINEAR_FUSED=$v timeout 300 python bench.py --workload decode > gpurun_out/s3_fx_${v}_${rep}.json 2> gpurun_out/s3_fx_${v}_${rep}.err
  done
done
