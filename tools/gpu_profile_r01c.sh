# Producer kernels and decode GEMMs: full captures (why are they far from the HBM roofline?)
mkdir -p gpurun_out
P="ncu --set full --clock-control none --import-source on"
REPS=3 timeout 300 $P -k regex:rmsnorm -s 2 -c 1 -o gpurun_out/r01_rms python tools/one_gemm.py rms 8192 4096 > gpurun_out/ncu_rms.log 2>&1; echo rms=$?
REPS=3 timeout 300 $P -k regex:silu -s 2 -c 1 -o gpurun_out/r01_silu python tools/one_gemm.py silu 8192 12288 > gpurun_out/ncu_silu.log 2>&1; echo silu=$?
REPS=3 timeout 300 $P -k regex:gemm -s 2 -c 1 -o gpurun_out/r01_dec1 python tools/one_gemm.py gemm 1 6144 4096 > gpurun_out/ncu_dec1.log 2>&1; echo dec1=$?
REPS=3 timeout 300 $P -k regex:gemm -s 2 -c 1 -o gpurun_out/r01_dec64 python tools/one_gemm.py gemm 64 6144 4096 > gpurun_out/ncu_dec64.log 2>&1; echo dec64=$?
REPS=3 timeout 300 $P -k regex:act_per_token -s 2 -c 1 -o gpurun_out/r01_aq_o python tools/one_gemm.py aq 8192 4096 > gpurun_out/ncu_aq.log 2>&1; echo aq=$?
ls gpurun_out
