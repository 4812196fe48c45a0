"""Fused one-kernel step vs the split step and the oracle (GPU quick check)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1405_6162_b200 as lk
from paper_1405_6162_b200.kernels import random_binary_state
from oracle import oracle as orc


def run(shape, kind, steps, seed=7, tau=(0.8, 1.1), mode=lk.MODE_EXACT, graph=True):
    f0, g0 = random_binary_state(lk.LatticeShape(*shape), np.random.default_rng(seed))
    model = lk.D3Q19Model(tau_f=tau[0], tau_g=tau[1])
    with lk.BinaryFluid(lk.LatticeShape(*shape), model=model, mode=mode, use_graph=graph) as sim:
        sim.set_step(kind)
        fused = sim.step_fused
        sim.load(f0, g0)
        sim.run(steps)
        f1, g1 = sim.fields()
        phi, mu = sim.order_parameter()
    return f0, g0, f1, g1, phi, mu, fused


ok = True
for shape, steps in [((32, 8, 4), 3), ((64, 6, 5), 4), ((32, 1, 7), 3), ((96, 16, 9), 5),
                     ((64, 64, 4), 2), ((128, 128, 32), 3)]:
    f0, g0, f1, g1, phi, mu, fz = run(shape, lk.STEP_FUSED, steps)
    _, _, f2, g2, phi2, mu2, fz2 = run(shape, lk.STEP_SPLIT, steps)
    same = (np.array_equal(f1.data.view(np.uint64), f2.data.view(np.uint64)) and
            np.array_equal(g1.data.view(np.uint64), g2.data.view(np.uint64)) and
            np.array_equal(phi, phi2) and np.array_equal(mu, mu2))
    prm = orc.fluid_params(tau_f=0.8, tau_g=1.1, physics=1)
    of, og, ophi, omu = orc.fluid_step(f0.data, g0.data, shape, f0.descriptor.padded_sites, prm,
                                       steps=steps, threads=16)
    orc_ok = np.array_equal(f1.data, of) and np.array_equal(g1.data, og) and \
        np.array_equal(phi.transpose(2, 1, 0).ravel(), ophi) and \
        np.array_equal(mu.transpose(2, 1, 0).ravel(), omu)
    if not (same and orc_ok):
        ok = False
        d = np.abs(f1.data - f2.data)
        print("  max|df| fused-split", d.max(), "phi", np.abs(phi - phi2).max(),
              "mu", np.abs(mu - mu2).max())
        bad = np.argwhere(np.abs(phi - phi2) > 0)[:10]
        print("  phi mismatch (z,y,x) first:", bad.tolist())
        badm = np.argwhere(np.abs(mu - mu2) > 0)[:10]
        print("  mu mismatch (z,y,x) first:", badm.tolist())
    print(shape, "fused" if fz else "NOT fused", fz2, "fused==split", same, "oracle", orc_ok,
          flush=True)

# K > 1 (more segments than resident warps)
for shape in [(256, 512, 4)]:
    _, _, f1, g1, phi, mu, fz = run(shape, lk.STEP_FUSED, 2, tau=(1.0, 1.0))
    _, _, f2, g2, phi2, mu2, _ = run(shape, lk.STEP_SPLIT, 2, tau=(1.0, 1.0))
    same = np.array_equal(f1.data, f2.data) and np.array_equal(g1.data, g2.data) and \
        np.array_equal(phi, phi2) and np.array_equal(mu, mu2)
    ok &= same
    print(shape, "K>1 fused==split", same, flush=True)

# timing 256^3
shape = lk.LatticeShape(256, 256, 256)
f0, g0 = random_binary_state(shape, np.random.default_rng(1234))
for kind in (lk.STEP_SPLIT, lk.STEP_FUSED):
    with lk.BinaryFluid(shape) as sim:
        sim.set_step(kind)
        sim.load(f0, g0)
        sim.run(3)
        sim.sync()
        import ctypes
        t = time.perf_counter()
        sim.run(20)
        sim.sync()
        dt = (time.perf_counter() - t) / 20
        print("256^3", "fused" if kind == lk.STEP_FUSED else "split", "%.4f ms/step" % (dt * 1e3),
              "%.0f MLUPS" % (shape.nsites / dt / 1e6), flush=True)
        if kind == lk.STEP_FUSED:
            ff, gf = sim.fields()
        else:
            fs, gs = sim.fields()
print("256^3 23 steps fused==split", np.array_equal(ff.data, fs.data) and np.array_equal(gf.data, gs.data))
print("ALL OK" if ok else "MISMATCH")
