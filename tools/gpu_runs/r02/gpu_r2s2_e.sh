# run E: the whole GPU suite after the exact producers / batched act quant / GEMM cleanup
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/e_gputests.txt
timeout 300 python tools/prod_bench.py > gpurun_out/e_prodbench.txt 2>&1
