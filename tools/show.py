import json, re
print(open('gpurun_out/gpu_tests.log').read().strip().splitlines()[-2:])
for f in ['bench_plm','bench_weno','bench_c3']:
    try:
        d=json.loads(open('gpurun_out/'+f+'.log').read().strip().splitlines()[-1])
        print(f, '%.4g zu/s'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], 'share %.3f'%d['roofline']['stage_kernel_share'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
    except Exception as e: print(f, e, open('gpurun_out/'+f+'.log').read()[-1500:])
