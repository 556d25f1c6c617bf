import json,sys,glob
for f in sorted(glob.glob(sys.argv[1])):
    try:
        d=json.load(open(f)); b=d['breakdown']
        print(f.split('/')[-1], d['value'], d['ms_per_step'], b['sync_ms'], b['requant_frac_hbm'], b['act_quant_ms'], b['act_quant_frac_hbm'], b['gemm_tflops'], d['clocks']['sm_mhz'])
    except Exception as e: print(f, 'ERR', e)
