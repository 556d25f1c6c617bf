# final check of the round's code: all GPU tests + smoke + a bench line
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_final.log 2>&1; echo tests=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo smoke=$?
tail -2 gpurun_out/gpu_tests_final.log; cat gpurun_out/smoke_final.log | tail -1
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench=$?
tail -1 gpurun_out/bench_final.json
