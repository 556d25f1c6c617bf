# run Z: decode layer, fused linear (XQ) vs two launches with the PDL-aware quantizer, same box
timeout 600 python bench.py --workload decode > gpurun_out/z_fused.json 2> gpurun_out/z_fused.err
FP8Q_LINEAR_FUSED=0 timeout 600 python bench.py --workload decode > gpurun_out/z_twostep.json 2> gpurun_out/z_twostep.err
