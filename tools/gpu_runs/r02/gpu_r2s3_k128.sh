# dev: one-CTA 128 x 128 tile kernel (4 TMEM buffers, 4 stages) for the MoE grouped GEMMs (FP8Q_GEMM_KIND=128) vs default 128 x 256
FP8Q_GEMM_KIND=128 timeout 900 python -m pytest tests/test_gpu_gemm.py -q -m gpu -k "grouped or moe" 2>&1 | tail -3 > gpurun_out/s3_k128_tests.txt
for rep in 1 2; do
  timeout 300 python bench.py --workload moe > gpurun_out/s3_k128_def_${rep}.json 2>gpurun_out/s3_k128_def_${rep}.err
  FP8Q_GEMM_KIND=128 timeout 300 python bench.py --workload moe > gpurun_out/s3_k128_128_${rep}.json 2>gpurun_out/s3_k128_128_${rep}.err
done
