# session-4 final evidence (HEAD: tail split incl. decode M = 256 dispatch): GPU suite, smoke, bench line, launch list with DRAM bytes, full captures
python paper_2601_18150_b200/build.py > gpurun_out/fin7_build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/fin7_gputests.txt
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/fin7_smoke.txt 2>&1
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/fin7_bench.json 2> gpurun_out/fin7_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin7_launches.csv python bench.py --steps 2 --warmup 1 --no-extras --no-e2e --no-cpu-baseline > gpurun_out/fin7_ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"pair_kernel|act_per_token|weight_blockwise_bulk|grouped|fp8_block_gemm_kernel" -c 8 -f -o gpurun_out/fin7_full python tools/prof_kernels.py > gpurun_out/fin7_ncu.txt 2>&1
