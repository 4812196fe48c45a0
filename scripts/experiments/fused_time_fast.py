"""Fused vs split step at 256^3 in FAST mode (timing only, GPU)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1405_6162_b200 as lk
from paper_1405_6162_b200.kernels import random_binary_state
shape = lk.LatticeShape(256, 256, 256)
f0, g0 = random_binary_state(shape, np.random.default_rng(1234))
out = {}
for mode in (lk.MODE_FAST, lk.MODE_EXACT):
    for kind in (lk.STEP_SPLIT, lk.STEP_FUSED):
        with lk.BinaryFluid(shape, mode=mode) as sim:
            sim.set_step(kind)
            sim.load(f0, g0)
            sim.run(3)
            sim.sync()
            t = time.perf_counter()
            sim.run(20)
            sim.sync()
            dt = (time.perf_counter() - t) / 20
            out[(mode, kind)] = sim.fields()
            print("mode", mode, "split" if kind == lk.STEP_SPLIT else "fused", "%.4f ms/step" % (dt * 1e3), flush=True)
    a, b = out[(mode, lk.STEP_SPLIT)], out[(mode, lk.STEP_FUSED)]
    print("  fused == split:", np.array_equal(a[0].data, b[0].data) and np.array_equal(a[1].data, b[1].data))
