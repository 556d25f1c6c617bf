# dev: weight quantizer bulk vs wide (host overhead hidden), decode GEMM graph timing, MoE
mkdir -p gpurun_out
echo "== pattern bulk"; timeout 300 python tools/pattern_bench.py | grep -v torch
echo "== pattern wide"; FP8Q_WEIGHT_KERNEL=wide timeout 300 python tools/pattern_bench.py | grep weight
echo "== kb wq bulk"; timeout 300 python tools/kernel_bench.py --what wq --flush read
echo "== kb wq wide"; FP8Q_WEIGHT_KERNEL=wide timeout 300 python tools/kernel_bench.py --what wq --flush read
echo "== decode"; timeout 600 python tools/kernel_bench.py --what none --decode --graph --flush read
echo "== moe"; timeout 600 python tools/kernel_bench.py --what none --moe --flush read
