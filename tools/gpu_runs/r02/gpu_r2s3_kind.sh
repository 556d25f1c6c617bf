# dev: decode GEMMs with the swap-AB kernel forced (FP8Q_GEMM_KIND=16) vs the default dispatch, graph timings
timeout 600 python tools/kernel_bench.py --what none --decode --graph --iters 10 > gpurun_out/s3_kind_def.txt 2>&1
FP8Q_GEMM_KIND=16 timeout 600 python tools/kernel_bench.py --what none --decode --graph --iters 10 > gpurun_out/s3_kind_16.txt 2>&1
