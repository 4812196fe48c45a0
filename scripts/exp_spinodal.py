"""Spinodal decomposition on the GPU (3-D validation of the builder-defined step):
a symmetric mixture phi = 0 +- 0.01 noise at the default free energy separates into
+-phi* domains that coarsen.  Every `every` steps: mean |phi|, the discrete free
energy F = sum(A/2 phi^2 + B/4 phi^4 + kappa/2 |grad phi|^2) (central gradient),
max |u|, and the dominant wavelength from the radially averaged structure factor.
Args: N steps every physics [mode].  Prints one JSON line."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1405_6162_b200 as lk  # noqa: E402
from paper_1405_6162_b200.lattice import FieldDescriptor, field_create  # noqa: E402

N, steps, every = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
physics = sys.argv[4]
mode = lk.MODE_EXACT if len(sys.argv) > 5 and sys.argv[5] == "exact" else lk.MODE_FAST
fe, model = lk.FreeEnergy(), lk.D3Q19Model()
shape = lk.LatticeShape(N, N, N)
desc = FieldDescriptor.create(19, shape.nsites)
f, g = field_create(desc), field_create(desc)
rng = np.random.default_rng(1405)
phi0 = 0.01 * (2 * rng.random(shape.nsites) - 1)
for i in range(19):
    f.component(i)[:] = model.wv[i]
    g.component(i)[:] = model.wv[i] * phi0
n, P = shape.nsites, desc.padded_sites
k = np.fft.fftfreq(N) * N
kk = np.sqrt(k[:, None, None] ** 2 + k[None, :, None] ** 2 + k[None, None, :] ** 2)
kbin = np.rint(kk).astype(int)
hist = []
with lk.BinaryFluid(shape, model=model, free_energy=fe, physics=physics, mode=mode) as sim:
    sim.load(f, g)
    for t in range(0, steps + 1, every):
        if t:
            sim.run(every)
        f1, g1 = sim.fields()
        F1 = f1.data.reshape(19, P)[:, :n]
        phi = g1.data.reshape(19, P)[:, :n].sum(0).reshape(N, N, N)
        u = (model.cvf.T @ F1) / F1.sum(0)
        grad = [(np.roll(phi, -1, a) - np.roll(phi, 1, a)) * 0.5 for a in range(3)]
        fen = float(np.sum(0.5 * fe.A * phi ** 2 + 0.25 * fe.B * phi ** 4
                           + 0.5 * fe.kappa * sum(gr * gr for gr in grad)))
        S = np.abs(np.fft.fftn(phi - phi.mean())) ** 2
        Sk = np.bincount(kbin.ravel(), S.ravel()) / np.maximum(np.bincount(kbin.ravel()), 1)
        kmax = int(np.argmax(Sk[1:N // 2]) + 1)
        ks = np.arange(len(Sk))
        tot = np.bincount(kbin.ravel(), S.ravel())
        kmean = float((ks[1:N // 2] * tot[1:N // 2]).sum() / max(tot[1:N // 2].sum(), 1e-300))
        hist.append({"t": t, "mean_abs_phi": float(np.abs(phi).mean()), "free_energy": fen,
                     "max_u": float(np.abs(u).max()), "wavelength": N / kmax,
                     "L": N / kmean if kmean > 0 else None,
                     "phi_sum": float(phi.sum()), "finite": bool(np.isfinite(F1).all())})
print(json.dumps({"N": N, "physics": physics, "mode": "exact" if mode == lk.MODE_EXACT else "fast",
                  "hist": hist}))
