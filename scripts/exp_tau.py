"""Collision-only (configs[1], 128^3) throughput at tau = 1.0 and 0.8 in both
arithmetic modes, through the latkit-compatible API.  Prints one line each."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1405_6162_b200 as lk  # noqa: E402
from paper_1405_6162_b200 import _native as nat  # noqa: E402
from paper_1405_6162_b200.kernels import random_binary_state  # noqa: E402

shape = lk.LatticeShape(128, 128, 128)
for tau in (1.0, 0.8):
    for mode, name in ((lk.MODE_EXACT, "exact"), (lk.MODE_FAST, "fast")):
        model = lk.D3Q19Model(tau_f=tau, tau_g=tau)
        f, g = random_binary_state(shape, np.random.default_rng(1234), model)
        dev = lk.TargetDevice()
        lk.set_model_constants(dev, model, mode)
        bf, bg = lk.target_malloc(dev, f.descriptor), lk.target_malloc(dev, g.descriptor)
        lk.copy_to_target(bf, f)
        lk.copy_to_target(bg, g)
        plan = lk.LaunchPlan(extent=f.descriptor.padded_sites, vvl=1, tpb=128)
        for _ in range(3):
            lk.launch(dev, lk.binary_collision_kernel, plan, [bf, bg])
        lk.sync_target(dev)
        a, b = nat.event_create(True), nat.event_create(True)
        n = 50
        nat.check(nat.lib.ltk_event_record(a, dev.stream))
        for _ in range(n):
            lk.launch(dev, lk.binary_collision_kernel, plan, [bf, bg])
        nat.check(nat.lib.ltk_event_record(b, dev.stream))
        lk.sync_target(dev)
        ms = nat.elapsed_ms(a, b) / n
        sites = shape.nsites
        print(f"collision 128^3 tau={tau} mode={name}: {sites / ms / 1e6:.2f} GLUPS "
              f"{608 * sites / ms / 1e6:.0f} GB/s", flush=True)
