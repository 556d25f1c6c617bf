# run V: GEMM operand ring 160 KB (base: pair 5 / one-CTA 3 stages) vs 192 KB (6 / 4 stages), same box
for i in 1 2; do
  FP8Q_LIB=$PWD/ab/libfp8q_base.so timeout 300 python tools/kernel_bench.py --what gemm --flush read > gpurun_out/v_base_$i.txt 2>&1
  timeout 300 python tools/kernel_bench.py --what gemm --flush read > gpurun_out/v_new_$i.txt 2>&1
done
FP8Q_LIB=$PWD/ab/libfp8q_base.so timeout 300 python tools/kernel_bench.py --what none --moe --flush read > gpurun_out/v_moe_base.txt 2>&1
timeout 300 python tools/kernel_bench.py --what none --moe --flush read > gpurun_out/v_moe_new.txt 2>&1
FP8Q_LIB=$PWD/ab/libfp8q_base.so timeout 300 python tools/shard_bench.py > gpurun_out/v_sh_base.txt 2>&1
timeout 300 python tools/shard_bench.py > gpurun_out/v_sh_new.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_gemm.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/v_tests.txt
