# session 3 baseline: restored tree -- GPU suite + default bench line
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/s3_base_smi.txt
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/s3_base_gputests.txt
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/s3_base_bench.json 2> gpurun_out/s3_base_bench.err
