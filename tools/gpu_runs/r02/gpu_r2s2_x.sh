# run X: operand-ring sensitivity -- 4 stages (ab/libfp8q_4stage.so) vs 5 (current), same box
for i in 1 2; do
  FP8Q_LIB=$PWD/ab/libfp8q_4stage.so timeout 300 python tools/kernel_bench.py --what gemm --flush read > gpurun_out/x_4st_$i.txt 2>&1
  timeout 300 python tools/kernel_bench.py --what gemm --flush read > gpurun_out/x_5st_$i.txt 2>&1
done
