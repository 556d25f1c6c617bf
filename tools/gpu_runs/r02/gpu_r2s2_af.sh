# run AF: ncu of the NEXT-2 producers (instruction mix / stalls)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"rmsnorm|silu_mul" -c 2 -o gpurun_out/af_prod python tools/prod_bench.py > gpurun_out/af_ncu.txt 2>&1
