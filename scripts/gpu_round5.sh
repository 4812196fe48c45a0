#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for m in fast exact; do
timeout 300 python bench.py --mode $m --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_$m.json 2>> gpurun_out/bench.err
done
python - > gpurun_out/tau_sweep.txt 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np
import paper_1405_6162_b200 as lk
from paper_1405_6162_b200.kernels import random_binary_state
shape = lk.LatticeShape(128, 128, 128)
for tau in (1.0, 0.8):
    for mode in (lk.MODE_EXACT, lk.MODE_FAST):
        r = lk.benchmark_run("binary-collision", shape, 1, iterations=50, mode=mode) if tau == 1.0 else None
        # tau != 1 through the API directly
        m = lk.D3Q19Model(tau_f=tau, tau_g=tau)
        f, g = random_binary_state(shape, np.random.default_rng(1234), m)
        dev = lk.TargetDevice(); lk.set_model_constants(dev, m, mode)
        bf, bg = lk.target_malloc(dev, f.descriptor), lk.target_malloc(dev, g.descriptor)
        lk.copy_to_target(bf, f); lk.copy_to_target(bg, g)
        plan = lk.LaunchPlan(extent=f.descriptor.padded_sites, vvl=1)
        from paper_1405_6162_b200 import _native as nat
        lk.launch(dev, lk.binary_collision_kernel, plan, [bf, bg]); lk.sync_target(dev)
        s, e = nat.event_create(True), nat.event_create(True)
        nat.lib.ltk_event_record(s, dev.stream)
        for _ in range(50): lk.launch(dev, lk.binary_collision_kernel, plan, [bf, bg])
        nat.lib.ltk_event_record(e, dev.stream); lk.sync_target(dev)
        ms = nat.elapsed_ms(s, e) / 50
        print(f"collision 128^3 tau={tau} mode={'exact' if mode == 0 else 'fast'}: {shape.nsites/ms/1e6:.2f} GLUPS {608*shape.nsites/ms/1e6:.0f} GB/s")
PY
