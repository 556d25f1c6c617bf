mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_quant.py tests/test_gpu_exhaustive.py tests/test_gpu_producers.py -x -q > gpurun_out/aq_tma_parity.log 2>&1; echo parity=$?
tail -1 gpurun_out/aq_tma_parity.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool racecheck --print-limit 5 python -m pytest tests/test_gpu_quant.py -x -q -m gpu -k "act" > gpurun_out/racecheck_aq_tma.log 2>&1; echo racecheck=$?
grep -E 'passed|failed|SUMMARY' gpurun_out/racecheck_aq_tma.log | tail -2
timeout 900 $CS --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_quant.py -x -q -m gpu -k "act" > gpurun_out/memcheck_aq_tma.log 2>&1; echo memcheck=$?
grep -E 'passed|failed|SUMMARY' gpurun_out/memcheck_aq_tma.log | tail -2
echo "== tma"; timeout 300 python tools/kernel_bench.py --what aq --flush read
echo "== bulk"; FP8Q_ACT_LOAD=bulk timeout 300 python tools/kernel_bench.py --what aq --flush read
timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tma layer', d['value'], d['breakdown']['act_quant_frac_hbm'])"
FP8Q_ACT_LOAD=bulk timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bulk layer', d['value'], d['breakdown']['act_quant_frac_hbm'])"
