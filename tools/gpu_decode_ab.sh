echo "== default"; timeout 600 python tools/kernel_bench.py --what none --decode --graph --flush read | grep -E '"shape": \[(64|128|256), 24576'
echo "== forced skinny"; FP8Q_GEMM_KIND=16 timeout 600 python tools/kernel_bench.py --what none --decode --graph --flush read | grep -E '"shape": \[(64|128|256), 24576'
