# dev: release-path timeline (debug 1) for the one-CTA and pair kernels
for kind in 256 1256; do
echo "== kind $kind"
FP8Q_GEMM_KIND=$kind FP8Q_GEMM_DEBUG=1 timeout 120 python tools/gemm_trace.py 8192 24576 4096 2>&1 | tail -13
done
