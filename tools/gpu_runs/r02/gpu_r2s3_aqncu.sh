# ncu full capture of the batched activation quantizer (one-vote build), source-level stalls
timeout 600 ncu --set full --import-source on --clock-control none -k regex:act_per_token_group_bulk -c 1 -f -o gpurun_out/s3_aq python tools/prof_kernels.py > gpurun_out/s3_aqncu.log 2>&1
