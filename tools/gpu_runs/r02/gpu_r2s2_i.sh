# run I: decode ring A/B (half vs full ring at M <= 32) + ncu full captures of the hot kernels
timeout 300 python tools/kernel_bench.py --what none --decode --graph --flush read > gpurun_out/i_kdec_half.txt 2>&1
FP8Q_SKINNY_RING=full timeout 300 python tools/kernel_bench.py --what none --decode --graph --flush read > gpurun_out/i_kdec_full.txt 2>&1
FP8Q_SKINNY_RING=full timeout 600 python bench.py --workload decode > gpurun_out/i_decode_full.json 2> gpurun_out/i_decode_full.err
timeout 900 ncu --set full --import-source on -k regex:"pair_kernel|act_per_token|grouped|fp8_block_gemm_kernel" -c 7 -o gpurun_out/i_full python tools/prof_kernels.py > gpurun_out/i_ncu.txt 2>&1
