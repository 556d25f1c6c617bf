# Round-1 evidence pass: launch list of one bench step, full captures of the three kernels.
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_r01.log 2>&1; echo ncu_launch=$?
REPS=3 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm -s 2 -c 1 -o gpurun_out/r01_gemm_qkv python tools/one_gemm.py gemm 8192 6144 4096 > gpurun_out/ncu_g1.log 2>&1; echo g1=$?
REPS=3 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm -s 2 -c 1 -o gpurun_out/r01_gemm_gateup python tools/one_gemm.py gemm 8192 24576 4096 > gpurun_out/ncu_g2.log 2>&1; echo g2=$?
REPS=3 timeout 300 ncu --set full --clock-control none --import-source on -k regex:weight_blockwise -s 2 -c 1 -o gpurun_out/r01_wq_gateup python tools/one_gemm.py wq 24576 4096 > gpurun_out/ncu_w.log 2>&1; echo wq=$?
REPS=3 timeout 300 ncu --set full --clock-control none --import-source on -k regex:act_per_token -s 2 -c 1 -o gpurun_out/r01_aq_down python tools/one_gemm.py aq 8192 12288 > gpurun_out/ncu_a.log 2>&1; echo aq=$?
REPS=3 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm -s 2 -c 1 -o gpurun_out/r01_grouped_fc1 python tools/one_gemm.py grouped 8192 gate_up > gpurun_out/ncu_g3.log 2>&1; echo g3=$?
ls -la gpurun_out
