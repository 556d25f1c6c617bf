# dev: A/B of the weight-quantizer path inside bench.py; decode per-CTA timelines
mkdir -p gpurun_out
for i in 1 2; do
for kind in auto wide; do
if [ $kind = wide ]; then export FP8Q_WEIGHT_KERNEL=wide; else unset FP8Q_WEIGHT_KERNEL; fi
timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown']; print('$kind', d['value'], b['sync_ms'], b['requant_frac_hbm'], b['gemm_tflops'], d['clocks']['sm_mhz'])"
done; done
unset FP8Q_WEIGHT_KERNEL
for mnk in "1 6144 4096" "64 6144 4096" "1 24576 4096"; do
echo "== trace $mnk"; timeout 120 python tools/skinny_trace.py $mnk 2>&1 | head -12
done
