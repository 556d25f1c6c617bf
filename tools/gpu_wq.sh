# dev: weight quantizer parity (incl. exhaustive map, fan-out) + timing, bulk vs wide
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_quant.py tests/test_gpu_exhaustive.py tests/test_gpu_fanout.py -x -q > gpurun_out/wq_parity.log 2>&1; echo parity=$?
tail -3 gpurun_out/wq_parity.log
echo "== bulk"; timeout 300 python tools/pattern_bench.py
echo "== wide"; FP8Q_WEIGHT_KERNEL=wide timeout 300 python tools/pattern_bench.py
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_wq.json 2> gpurun_out/bench_wq.err; echo bench=$?
tail -1 gpurun_out/bench_wq.json
