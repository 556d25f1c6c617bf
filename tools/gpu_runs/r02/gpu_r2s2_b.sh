# run B: batched activation quantizer parity + the default bench line
timeout 900 python -m pytest tests/test_gpu_quant.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/b_quant.txt
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err
