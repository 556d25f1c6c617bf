# run 3C: ordered stream-K for the decode kernel -- GEMM/linear GPU tests, decode layer A/B vs the atomic fixup, timeline
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_linear.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/c3_tests.txt
for cfg in "ord:1" "atomic:0" "ord2:1" "atomic2:0"; do
  IFS=: read name fl <<< "$cfg"
  FP8Q_SKINNY_ORDERED=$fl timeout 600 python bench.py --workload decode > gpurun_out/c3_$name.json 2> gpurun_out/c3_$name.err
done
timeout 300 python tools/decode_timeline.py --m 1 > gpurun_out/c3_tl_m1.txt 2>&1
FP8Q_SKINNY_ORDERED=1 FP8Q_SKINNY_TRIGGER=late timeout 600 python bench.py --workload decode > gpurun_out/c3_ordlate.json 2> gpurun_out/c3_ordlate.err
