mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_quant.py tests/test_gpu_exhaustive.py -x -q -k "act" > gpurun_out/aqcfg.log 2>&1; echo parity=$?; tail -1 gpurun_out/aqcfg.log
timeout 300 python tools/kernel_bench.py --what aq --flush read
timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('layer', d['value'], d['breakdown']['act_quant_frac_hbm'])"
