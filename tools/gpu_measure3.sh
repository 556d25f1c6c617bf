# dev: weight quantizer parity (forced paths) + bench; decode timelines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_quant.py tests/test_gpu_fanout.py -x -q > gpurun_out/wq_parity.log 2>&1; echo parity=$?
tail -3 gpurun_out/wq_parity.log
echo "== kb wq"; timeout 300 python tools/kernel_bench.py --what wq --flush write
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_wq.json 2> gpurun_out/bench_wq.err; echo bench=$?
tail -1 gpurun_out/bench_wq.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['breakdown'])"
for mnk in "1 6144 4096" "64 6144 4096" "1 24576 4096"; do
echo "== trace $mnk"; timeout 120 python tools/skinny_trace.py $mnk | head -30
echo "== trace pair $mnk"; timeout 120 python tools/skinny_trace.py $mnk --pair | head -8
done
