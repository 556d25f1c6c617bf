# session 4: source-level ncu capture of the MoE fc2 grouped GEMM (one-CTA kernel), for the per-tile boundary cost
python paper_2601_18150_b200/build.py > gpurun_out/s4i_build.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fp8_block_gemm_kernel" -c 1 -f -o gpurun_out/s4i_fc2 python tools/prof_kernels.py > gpurun_out/s4i_ncu.txt 2>&1
ncu -i gpurun_out/s4i_fc2.ncu-rep --page source --csv --print-source sass > gpurun_out/s4i_src_sass.csv 2>/dev/null
ncu -i gpurun_out/s4i_fc2.ncu-rep --page source --csv --print-source cuda > gpurun_out/s4i_src_cuda.csv 2>/dev/null
