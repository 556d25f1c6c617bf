mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool racecheck --print-limit 5 python -m pytest tests/test_gpu_quant.py -x -q -m gpu -k "act" > gpurun_out/racecheck_aq.log 2>&1; echo racecheck_aq=$?
grep -E 'passed|failed|SUMMARY|Race reported' gpurun_out/racecheck_aq.log | head -5
timeout 900 python -m pytest tests/test_gpu_exhaustive.py -x -q -k activation > gpurun_out/exh_aq.log 2>&1; echo exhaustive=$?; tail -1 gpurun_out/exh_aq.log
timeout 300 python tools/kernel_bench.py --what aq --flush read
