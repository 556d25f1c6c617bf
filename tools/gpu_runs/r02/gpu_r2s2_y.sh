# run Y: PDL-aware activation quantizers (register path for <= 256 tokens) -- parity + decode layer
timeout 1200 python -m pytest tests/test_gpu_quant.py tests/test_gpu_linear.py tests/test_gpu_exhaustive.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/y_tests.txt
timeout 600 python bench.py --workload decode > gpurun_out/y_decode.json 2> gpurun_out/y_decode.err
FP8Q_LIB=$PWD/ab/libfp8q_base.so timeout 600 python bench.py --workload decode > gpurun_out/y_decode_base.json 2> gpurun_out/y_decode_base.err
