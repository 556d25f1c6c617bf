# dev A/B: e2e pipeline row blocks per GEMM (FP8Q_E2E_CHUNKS), 4 interleaved reps
for rep in 1 2 3 4; do
  for c in 4 16; do
    FP8Q_E2E_CHUNKS=$c timeout 300 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/s3_e2e_${c}_${rep}.json 2> /dev/null
  done
done
