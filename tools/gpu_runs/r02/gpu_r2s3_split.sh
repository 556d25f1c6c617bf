# dev: one-CTA tile kernel with split-K at decode M (coalesced [tile][split][col][row] partials) via FP8Q_GEMM_KIND=256 FP8Q_SPLIT_MAXM=256, vs the default dispatch
timeout 600 python tools/kernel_bench.py --what none --decode --graph --iters 10 > gpurun_out/s3_split_def.txt 2>&1
FP8Q_GEMM_KIND=256 FP8Q_SPLIT_MAXM=256 timeout 600 python tools/kernel_bench.py --what none --decode --graph --iters 10 > gpurun_out/s3_split_k256.txt 2>&1

