# run U: TP shard shapes, CTA-pair (1256) vs one-CTA (256) tiles
FP8Q_GEMM_KIND=1256 timeout 300 python tools/shard_bench.py > gpurun_out/u_1256.txt 2>&1
FP8Q_GEMM_KIND=256 timeout 300 python tools/shard_bench.py > gpurun_out/u_256.txt 2>&1
