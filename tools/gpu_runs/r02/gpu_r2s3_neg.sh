# A/B: negated Markstein encode (no input-sign gather) in the quantizers' element map (new) vs HEAD (base)
timeout 1200 python -m pytest tests -m gpu -q -x -k "quant or exhaustive or sync or fanout or smoke" 2>&1 | tail -3 > gpurun_out/s3_neg_tests.txt
for rep in 1 2 3; do
  for lib in base new; do
    if [ $lib = base ]; then export FP8Q_LIB=$PWD/paper_2601_18150_b200/libfp8q_base.so; else unset FP8Q_LIB; fi
    timeout 300 python bench.py --steps 20 --warmup 5 --no-extras --no-e2e --no-cpu-baseline > gpurun_out/s3_neg_${lib}_${rep}.json 2> /dev/null
  done
done
