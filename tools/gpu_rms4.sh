mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_producers.py -x -q > gpurun_out/prod_parity.log 2>&1; echo parity=$?; tail -1 gpurun_out/prod_parity.log
timeout 600 python tools/kernel_bench.py --what prod --flush read
