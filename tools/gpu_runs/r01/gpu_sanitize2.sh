# compute-sanitizer over the kernels added late in round 1: the TMA-staged weight quantizer
# (forced on every small shape) and the decode kernel's cluster split-K (DSMEM reduction)
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
K="not exhaustive and not full and not 8192 and not forced_path"
FP8Q_WEIGHT_KERNEL=bulk timeout 900 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_quant.py tests/test_gpu_fanout.py -x -q -m gpu -k "$K" > gpurun_out/memcheck_wq_bulk.log 2>&1; echo memcheck_wq_bulk=$?
FP8Q_WEIGHT_KERNEL=bulk timeout 900 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_quant.py -x -q -m gpu -k "$K" > gpurun_out/racecheck_wq_bulk.log 2>&1; echo racecheck_wq_bulk=$?
timeout 900 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_gemm.py -x -q -m gpu -k "skinny_decode_vs_oracle" > gpurun_out/memcheck_skinny.log 2>&1; echo memcheck_skinny=$?
timeout 900 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_gemm.py -x -q -m gpu -k "skinny_decode_vs_oracle" > gpurun_out/racecheck_skinny.log 2>&1; echo racecheck_skinny=$?
for f in memcheck_wq_bulk racecheck_wq_bulk memcheck_skinny racecheck_skinny; do echo "== $f"; grep -E 'passed|failed|SUMMARY' gpurun_out/$f.log | tail -3; done
