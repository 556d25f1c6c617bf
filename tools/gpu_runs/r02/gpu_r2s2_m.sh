# run M: A/B on one box -- committed GEMM (base) vs branch-free scale loads + predicated releases
for i in 1 2; do
  FP8Q_LIB=$PWD/ab/libfp8q_base.so FP8Q_GEMM_KIND=1256 timeout 300 python tools/kernel_bench.py --what gemm --flush read > gpurun_out/m_base_$i.txt 2>&1
  FP8Q_GEMM_KIND=1256 timeout 300 python tools/kernel_bench.py --what gemm --flush read > gpurun_out/m_new_$i.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_gemm.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/m_tests.txt
