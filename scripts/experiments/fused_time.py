"""Fused vs split step at 256^3: parity on two small shapes, then timing (GPU)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1405_6162_b200 as lk
from paper_1405_6162_b200.kernels import random_binary_state

nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
kinds = sys.argv[2].split(",") if len(sys.argv) > 2 else ["split", "fused"]
K = {"split": lk.STEP_SPLIT, "fused": lk.STEP_FUSED}
for shape in [(32, 8, 4), (96, 16, 9), (128, 128, 32)]:
    res = {}
    f0, g0 = random_binary_state(lk.LatticeShape(*shape), np.random.default_rng(3))
    for kind in ("split", "fused"):
        with lk.BinaryFluid(lk.LatticeShape(*shape), model=lk.D3Q19Model(tau_f=0.8, tau_g=1.1)) as sim:
            sim.set_step(K[kind])
            sim.load(f0, g0)
            sim.run(5)
            res[kind] = sim.fields() + sim.order_parameter()
    same = all(np.array_equal(np.asarray(getattr(a, "data", a)), np.asarray(getattr(b, "data", b)))
               for a, b in zip(res["split"], res["fused"]))
    print(shape, "fused == split:", same, flush=True)
shape = lk.LatticeShape(256, 256, 256)
f0, g0 = random_binary_state(shape, np.random.default_rng(1234))
for kind in kinds:
    with lk.BinaryFluid(shape) as sim:
        sim.set_step(K[kind])
        sim.load(f0, g0)
        sim.run(3)
        sim.sync()
        sim.profile(True)
        t = time.perf_counter()
        sim.run(nsteps)
        sim.sync()
        dt = (time.perf_counter() - t) / nsteps
        ms = sim.profile(False)
        print("256^3 %s: %.4f ms/step wall, %.0f MLUPS; per step phi %.4f mu %.4f cs %.4f total %.4f ms"
              % (kind, dt * 1e3, shape.nsites / dt / 1e6, ms[0] / nsteps, ms[1] / nsteps,
                 ms[2] / nsteps, ms[3] / nsteps), flush=True)
