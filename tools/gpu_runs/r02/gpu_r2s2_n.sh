# run N: evidence checkpoint (whole GPU suite, default bench line, launch list) + PDL on/off decode A/B
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -6 > gpurun_out/n_gputests.txt
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/n_bench.json 2> gpurun_out/n_bench.err
timeout 300 python tools/kernel_bench.py --what none --decode --graph --flush read > gpurun_out/n_kdec_pdl.txt 2>&1
FP8Q_SKINNY_NOPDL=1 timeout 300 python tools/kernel_bench.py --what none --decode --graph --flush read > gpurun_out/n_kdec_nopdl.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/n_launches.csv python bench.py --steps 2 --warmup 1 --no-extras --no-e2e --no-cpu-baseline > gpurun_out/n_ncu_bench.log 2>&1
