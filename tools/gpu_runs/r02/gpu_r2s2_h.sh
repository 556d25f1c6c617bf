# run H: XQ after the padding / zero-group fix
timeout 300 python tools/xq_probe.py > gpurun_out/h_probe.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_linear.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/h_tests.txt
timeout 600 python bench.py --workload decode > gpurun_out/h_decode.json 2> gpurun_out/h_decode.err
