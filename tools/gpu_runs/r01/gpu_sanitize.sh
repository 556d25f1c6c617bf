# compute-sanitizer memcheck / racecheck over small instances of every kernel family
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_gpu_quant.py tests/test_gpu_producers.py tests/test_gpu_kv.py tests/test_gpu_fanout.py"
timeout 900 $CS --tool memcheck --print-limit 20 python -m pytest $T -x -q -m gpu -k "not exhaustive and not full and not 8192" > gpurun_out/memcheck_quant.log 2>&1; echo memcheck_quant=$?
timeout 900 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_mx.py -x -q -m gpu -k "small or probe or skinny or grouped_vs or decode_vs or quantize_bit" > gpurun_out/memcheck_gemm.log 2>&1; echo memcheck_gemm=$?
timeout 900 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_quant.py tests/test_gpu_producers.py -x -q -m gpu -k "not exhaustive and not full and not 8192" > gpurun_out/racecheck_quant.log 2>&1; echo racecheck_quant=$?
tail -4 gpurun_out/memcheck_quant.log gpurun_out/memcheck_gemm.log gpurun_out/racecheck_quant.log
