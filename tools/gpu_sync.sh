# whole-model weight sync at P = 1 (C5 / the 8B analogue): requant of every linear weight per step
mkdir -p gpurun_out
for wl in sync8b sync30b; do
timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err; echo $wl=$?
tail -1 gpurun_out/bench_$wl.json
FP8Q_WEIGHT_KERNEL=wide timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('wide', d['value'], d.get('roofline'))"
done
