set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_gpu_sync.py tests/test_gpu_fullsize.py -q -x -m gpu 2>&1 | tail -30 > gpurun_out/r2_newtests.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err
tail -5 gpurun_out/r2_bench1.err
cat gpurun_out/r2_newtests.txt
