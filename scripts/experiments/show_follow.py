import json, csv, sys
cfg = None
for ln in open('gpurun_out/bench_follow.txt'):
    if ln.startswith('=='): cfg = ln.strip(); continue
    if ln.startswith('{'):
        d = json.loads(ln); r = d['roofline']
        print(cfg, 'ms/step %.4f' % d['ms_per_step'], 'MLUPS %.0f' % d['value'], 'cs %.4f' % r['kernel_ms_per_step'],
              'phi %.4f mu %.4f' % (r['phi_ms_per_step'], r['mu_ms_per_step']), 'drift', d['conservation']['mass_rel_drift'])
    elif 'rror' in ln: print(ln.strip()[:200])
try:
    for r in csv.reader(open('gpurun_out/ncu_range_f1.csv')):
        if len(r) > 10 and r[4] == 'range': print(r[10], r[12])
except Exception as e: print(e)
