# run K: MoE grouped GEMM, one-CTA (256) vs CTA-pair (1256) tiles after the dev-branch removal
FP8Q_GEMM_KIND=256 timeout 600 python tools/kernel_bench.py --what none --moe --flush read > gpurun_out/k_moe_256.txt 2>&1
FP8Q_GEMM_KIND=1256 timeout 600 python tools/kernel_bench.py --what none --moe --flush read > gpurun_out/k_moe_1256.txt 2>&1
