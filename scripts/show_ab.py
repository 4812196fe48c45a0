import json
cfg = None
for ln in open('gpurun_out/ab.txt'):
    if ln.startswith('=='): cfg = ln.strip(); continue
    if ln.startswith('{'):
        d = json.loads(ln); r = d['roofline']
        print(f"{cfg:50s} ms/step {d['ms_per_step']:.4f} MLUPS {d['value']:.0f} cs {r['kernel_ms_per_step']:.4f} phi {r['phi_ms_per_step']:.4f} mu {r['mu_ms_per_step']:.4f} launches {d['gpu_launches']}")
    elif 'rror' in ln: print(ln.strip()[:200])
