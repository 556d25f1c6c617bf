# A/B: act quant TMA path without load masks (new) vs HEAD (base)
timeout 900 python -m pytest tests -m gpu -q -x -k "quant or exhaustive or sync" 2>&1 | tail -3 > gpurun_out/s3_nm_tests.txt
for rep in 1 2 3; do
  for lib in base new; do
    if [ $lib = base ]; then export FP8Q_LIB=$PWD/paper_2601_18150_b200/libfp8q_base.so; else unset FP8Q_LIB; fi
    timeout 300 python bench.py --steps 20 --warmup 5 --no-extras --no-e2e --no-cpu-baseline > gpurun_out/s3_nm_${lib}_${rep}.json 2> gpurun_out/s3_nm_${lib}_${rep}.err
    timeout 300 python tools/kernel_bench.py --what aq --iters 20 > gpurun_out/s3_nmk_${lib}_${rep}.txt 2>&1
  done
done
