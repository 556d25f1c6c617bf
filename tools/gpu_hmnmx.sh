# dev: HMNMX2 amax -- quantizer parity (incl. exhaustive + non-finite), timing, sync
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_quant.py tests/test_gpu_exhaustive.py tests/test_gpu_fanout.py -x -q > gpurun_out/q_parity.log 2>&1; echo parity=$?
tail -2 gpurun_out/q_parity.log
timeout 300 python tools/pattern_bench.py | grep -v torch
timeout 300 python tools/kernel_bench.py --what wq --flush read
timeout 300 python tools/kernel_bench.py --what aq --flush read
timeout 900 python bench.py --workload sync30b --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sync30b', d['value'], d['roofline']['frac'])"
timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('layer', d['value'], d['breakdown'])"
