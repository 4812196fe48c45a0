#!/bin/bash
# quick bench line (no e2e / cpu / config1) + optional extra command
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 120 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-config1 > gpurun_out/quick.json 2> gpurun_out/quick.err
python - <<'PY'
import json
d = json.loads(open('gpurun_out/quick.json').read().strip().splitlines()[-1]); r = d['roofline']
print('ms/step %.4f MLUPS %.0f cs %.4f phi %.4f mu %.4f frac %.3f' % (d['ms_per_step'], d['value'], r['kernel_ms_per_step'], r['phi_ms_per_step'], r['mu_ms_per_step'], r['frac']))
PY
