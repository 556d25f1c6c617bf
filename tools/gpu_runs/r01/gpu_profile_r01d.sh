# Round-1 evidence for the kernels added after r01: decode GEMM (swap-AB + stream-K),
# NEXT-2 producers, NEXT-3 KV append.  Full captures, one launch each.
mkdir -p gpurun_out
P="ncu --set full --clock-control none --import-source on"
REPS=3 timeout 300 $P -k regex:skinny -s 2 -c 1 -o gpurun_out/r01_dec1_skinny python tools/one_gemm.py gemm 1 6144 4096 > /dev/null 2>&1; echo dec1=$?
REPS=3 timeout 300 $P -k regex:skinny -s 2 -c 1 -o gpurun_out/r01_dec64_skinny python tools/one_gemm.py gemm 64 4096 12288 > /dev/null 2>&1; echo dec64=$?
REPS=3 timeout 300 $P -k regex:rmsnorm -s 2 -c 1 -o gpurun_out/r01_rms_fixed python tools/one_gemm.py rms 8192 4096 > /dev/null 2>&1; echo rms=$?
REPS=3 timeout 300 $P -k regex:silu -s 2 -c 1 -o gpurun_out/r01_silu_packed python tools/one_gemm.py silu 8192 12288 > /dev/null 2>&1; echo silu=$?
REPS=3 timeout 300 $P -k regex:kv_append -s 2 -c 1 -o gpurun_out/r01_kv_append python tools/one_gemm.py kv 8192 1024 > /dev/null 2>&1; echo kv=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
ls gpurun_out
