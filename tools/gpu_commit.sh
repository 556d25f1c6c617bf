mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q -k "not skinny and not grouped" > gpurun_out/gemm_parity.log 2>&1; echo parity=$?
tail -1 gpurun_out/gemm_parity.log
timeout 300 python tools/kernel_bench.py --what gemm --flush read 2>&1 | grep TFLOP
git_stash_note="(compare: 1256 before = 1917/1912/2101/2108 and 1899/1890/2070/2097 on earlier boxes)"
echo $git_stash_note
