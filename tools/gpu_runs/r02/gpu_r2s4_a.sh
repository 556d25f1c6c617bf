# session-4 re-entry: GPU suite + smoke + bench on the restored tree; decode GEMMs default vs forced swap-AB
python paper_2601_18150_b200/build.py > gpurun_out/s4a_build.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/s4a_gputests.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s4a_smoke.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s4a_bench.json 2> gpurun_out/s4a_bench.err
timeout 600 python tools/kernel_bench.py --what none --decode --graph --iters 10 > gpurun_out/s4a_kind_def.txt 2>&1
FP8Q_GEMM_KIND=16 timeout 600 python tools/kernel_bench.py --what none --decode --graph --iters 10 > gpurun_out/s4a_kind_16.txt 2>&1
