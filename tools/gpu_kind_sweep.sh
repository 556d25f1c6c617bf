# dev: parity of a forced GEMM kind on the GEMM tests + per-shape timing of several kinds
mkdir -p gpurun_out
KINDS=${KINDS:-"1256 2256 1128"}
FP8Q_GEMM_KIND=${PARITY_KIND:-2256} timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/kind_parity.log 2>&1; echo parity=$?
tail -3 gpurun_out/kind_parity.log
for k in $KINDS; do
  echo "kind $k"
  FP8Q_GEMM_KIND=$k timeout 300 python tools/kernel_bench.py --what gemm --iters 30 2>&1 | tee gpurun_out/kind_$k.jsonl | python -c "
import sys, json
for l in sys.stdin:
    try: r = json.loads(l)
    except Exception: print(l.strip()); continue
    print(r['shape'], r['ms'], r['TFLOPs'], r['frac_fp8'])"
done
