# Round-1 evidence refresh after the TMA-staged weight quantizer and the decode cluster split-K:
# gpu tests, smoke, bench line, launch list, full captures of the changed kernels, MoE kind A/B.
mkdir -p gpurun_out
bash tools/gpu_full_round.sh
P="ncu --set full --clock-control none --import-source on"
REPS=3 timeout 300 $P -k regex:weight_blockwise_bulk -s 2 -c 1 -o gpurun_out/r01_wq_layer_tma python tools/one_gemm.py wqlayer > /dev/null 2>&1; echo wq=$?
REPS=3 timeout 300 $P -k regex:skinny -s 2 -c 1 -o gpurun_out/r01_dec1_o_cluster python tools/one_gemm.py gemm 1 4096 4096 > /dev/null 2>&1; echo dec1=$?
REPS=3 timeout 300 $P -k regex:skinny -s 2 -c 1 -o gpurun_out/r01_dec128_o_cluster python tools/one_gemm.py gemm 128 4096 4096 > /dev/null 2>&1; echo dec128=$?
echo "== moe default"; timeout 600 python tools/kernel_bench.py --what none --moe --flush read | grep 8192
echo "== moe kind 128"; FP8Q_GEMM_KIND=128 timeout 600 python tools/kernel_bench.py --what none --moe --flush read | grep 8192
