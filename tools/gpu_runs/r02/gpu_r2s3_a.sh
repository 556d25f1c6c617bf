# run 3A: decode layer A/B -- trigger the dependent launch late (after the last TMA issue) and
# warm L2 with the next weight tiles before griddepcontrol.wait; parity of the decode tests first
set -x
FP8Q_SKINNY_TRIGGER=late FP8Q_SKINNY_L2PF=16 timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_linear.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/a3_tests.txt
for cfg in "base::" "late:late:" "pf8::8" "pf16::16" "pf32::32" "late_pf8:late:8" "late_pf16:late:16" "late_pf32:late:32" "base2::"; do
  IFS=: read name trig pf <<< "$cfg"
  FP8Q_SKINNY_TRIGGER=$trig FP8Q_SKINNY_L2PF=$pf timeout 600 python bench.py --workload decode > gpurun_out/a3_$name.json 2> gpurun_out/a3_$name.err
done
python - <<'PY' > gpurun_out/a3_summary.txt
import json, glob
for f in sorted(glob.glob("gpurun_out/a3_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    rec = d.get("decode", d)
    print(f, json.dumps(rec)[:900])
PY
