# dev: activation quantizer parity (incl. exhaustive map) + timing, bulk vs wide
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_quant.py tests/test_gpu_exhaustive.py -x -q > gpurun_out/aq_parity.log 2>&1; echo parity=$?
tail -3 gpurun_out/aq_parity.log
for fl in read; do
echo "== flush $fl bulk"; timeout 300 python tools/kernel_bench.py --what aq --iters 30 --flush $fl
echo "== flush $fl wide"; FP8Q_ACT_KERNEL=wide timeout 300 python tools/kernel_bench.py --what aq --iters 30 --flush $fl
done
