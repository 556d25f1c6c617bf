# ncu full captures (source-level stalls) of the staged weight quantizer (layer batch) and the batched activation quantizer
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"weight_blockwise_bulk|act_per_token_group_bulk" -c 2 -f -o gpurun_out/s3_q python tools/prof_kernels.py > gpurun_out/s3_qncu.log 2>&1
