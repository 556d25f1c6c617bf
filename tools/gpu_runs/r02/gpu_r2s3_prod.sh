# producer-fused quantizers: timing + ncu full capture of rmsnorm_quantize (source-level)
timeout 300 python tools/prod_bench.py > gpurun_out/s3_prod.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"rmsnorm_quantize|silu_mul_quantize_kernel" -c 2 -f -o gpurun_out/s3_prod python tools/prod_bench.py > gpurun_out/s3_prod_ncu.log 2>&1
