# A/B: producer-fused quantizers, y = ONE bf16x2 multiply where exact (binary32 fallback otherwise) (new) vs HEAD (base)
timeout 1200 python -m pytest tests -m gpu -q -x -k "producer or rmsnorm or silu" 2>&1 | tail -3 > gpurun_out/s3_prod3_tests.txt
for rep in 1 2; do
  for lib in base new; do
    if [ $lib = base ]; then export FP8Q_LIB=$PWD/paper_2601_18150_b200/libfp8q_base.so; else unset FP8Q_LIB; fi
    timeout 300 python tools/prod_bench.py > gpurun_out/s3_prod3_${lib}_${rep}.txt 2>&1
  done
done
