mkdir -p gpurun_out
set -x
nproc
timeout 300 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench_rc=$?
tail -3 gpurun_out/bench1.err
cat gpurun_out/bench1.json
timeout 900 python -m pytest tests/test_gpu_exhaustive.py -x -q -m gpu > gpurun_out/exh.log 2>&1; echo exh_rc=$?; tail -5 gpurun_out/exh.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fp8_block_gemm -s 13 -c 4 -o gpurun_out/prof_gemm python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1; echo ncu2_rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"weight_blockwise|act_per_token" -s 8 -c 8 -o gpurun_out/prof_quant python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_quant.log 2>&1; echo ncu3_rc=$?
ls -la gpurun_out
