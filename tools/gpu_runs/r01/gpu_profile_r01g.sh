# final round-1 evidence: full captures of the final quantizers, gpu tests, smoke, bench, launch list
mkdir -p gpurun_out
P="ncu --set full --clock-control none --import-source on"
REPS=3 timeout 300 $P -k regex:act_per_token -s 2 -c 1 -o gpurun_out/r01_aq_tma_4096 python tools/one_gemm.py aq 8192 4096 > /dev/null 2>&1; echo aq=$?
REPS=3 timeout 300 $P -k regex:act_per_token -s 2 -c 1 -o gpurun_out/r01_aq_tma_12288 python tools/one_gemm.py aq 8192 12288 > /dev/null 2>&1; echo aq2=$?
bash tools/gpu_full_round.sh
