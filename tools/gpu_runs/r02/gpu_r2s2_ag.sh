# run AG: ncu of a small-N shard GEMM ([8192, 512, 4096], o_proj at P = 8): why it runs at half the per-k-block rate
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pair_kernel --launch-skip 4 -c 1 -o gpurun_out/ag_shard python tools/shard_bench.py > gpurun_out/ag_ncu.txt 2>&1
