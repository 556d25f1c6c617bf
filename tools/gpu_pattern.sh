# dev: streaming-pattern ceiling vs the quantizers; full ncu capture of the bulk activation quantizer
mkdir -p gpurun_out
timeout 300 python tools/pattern_bench.py > gpurun_out/pattern.txt 2>&1; echo pattern=$?
P="ncu --set full --clock-control none --import-source on"
REPS=3 timeout 300 $P -k regex:act_per_token -s 2 -c 1 -o gpurun_out/r01_aq_bulk_4096 python tools/one_gemm.py aq 8192 4096 > /dev/null 2>&1; echo aq=$?
REPS=3 timeout 300 $P -k regex:weight_block -s 2 -c 1 -o gpurun_out/r01_wq_24576 python tools/one_gemm.py wq 24576 4096 > /dev/null 2>&1; echo wq=$?
cat gpurun_out/pattern.txt
