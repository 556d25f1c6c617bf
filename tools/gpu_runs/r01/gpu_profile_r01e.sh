# NEXT-4 MXFP8 GEMM vs the fp32-scale promotion kernel on the same shape (qkv, M = 8192)
mkdir -p gpurun_out
P="ncu --set full --clock-control none --import-source on"
REPS=3 timeout 300 $P -k regex:mx_gemm -s 2 -c 1 -o gpurun_out/r01_mx_qkv python tools/one_gemm.py mxgemm 8192 6144 4096 > /dev/null 2>&1; echo mx=$?
REPS=3 timeout 300 $P -k regex:mx_quantize -s 2 -c 1 -o gpurun_out/r01_mxq python tools/one_gemm.py mxgemm 8192 6144 4096 > /dev/null 2>&1; echo mxq=$?
REPS=3 timeout 300 $P -k regex:gemm -s 2 -c 1 -o gpurun_out/r01_pair_qkv python tools/one_gemm.py gemm 8192 6144 4096 > /dev/null 2>&1; echo pair=$?
ls gpurun_out | grep r01_
