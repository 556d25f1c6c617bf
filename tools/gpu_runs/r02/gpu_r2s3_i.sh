# run 3I: activation quantizer -- isolated timings vs torch's bf16->e4m3 cast, and one ncu --set full capture (source page) of the staged kernel
timeout 300 python tools/kernel_bench.py --what aq > gpurun_out/i3_aq.txt 2>&1
timeout 300 python tools/kernel_bench.py --what aqref > gpurun_out/i3_aqref.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:act_per_token_group_bulk --launch-skip 30 -c 1 -o gpurun_out/i3_aq python tools/kernel_bench.py --what aq --iters 5 > gpurun_out/i3_ncu.log 2>&1
