"""History of the flat double interface: max |u| and bulk phi every `every` steps
(see exp_interface.py).  Args: NXxNYxNZ steps every A B kappa gamma tau_f tau_g."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1405_6162_b200 as lk  # noqa: E402
from paper_1405_6162_b200.lattice import FieldDescriptor, field_create  # noqa: E402

nx, ny, nz = (int(v) for v in sys.argv[1].split("x"))
steps, every = int(sys.argv[2]), int(sys.argv[3])
A, B, kappa, gamma, tau_f, tau_g = map(float, sys.argv[4:10])
physics = sys.argv[10] if len(sys.argv) > 10 else "binary"
fe = lk.FreeEnergy(A=A, B=B, kappa=kappa, gamma=gamma)
model = lk.D3Q19Model(tau_f=tau_f, tau_g=tau_g)
shape = lk.LatticeShape(nx, ny, nz)
desc = FieldDescriptor.create(19, shape.nsites)
f, g = field_create(desc), field_create(desc)
z = np.arange(nz)
xi = np.sqrt(-2 * kappa / A)
prof0 = np.tanh((z - nz / 4 + 0.5) / xi) * np.tanh((3 * nz / 4 - 0.5 - z) / xi)
phi0 = np.broadcast_to(prof0, (nx, ny, nz)).reshape(-1)
for i in range(19):
    f.component(i)[:] = model.wv[i]
    g.component(i)[:] = model.wv[i] * phi0
n, P = shape.nsites, desc.padded_sites
cv = model.cvf
hist = []
with lk.BinaryFluid(shape, model=model, free_energy=fe, mode=lk.MODE_FAST, physics=physics) as sim:
    sim.load(f, g)
    for t in range(0, steps + 1, every):
        if t:
            sim.run(every)
        f1, g1 = sim.fields()
        F = f1.data.reshape(19, P)[:, :n]
        G = g1.data.reshape(19, P)[:, :n]
        rho = F.sum(0)
        uz = (cv[:, 2][:, None] * F).sum(0) / rho
        phi = G.sum(0)
        hist.append([t, float(np.abs(uz).max()), float(phi.max()), float(rho.max() - rho.min())])
print(json.dumps({"physics": physics, "A": A, "B": B, "kappa": kappa, "gamma": gamma, "tau_f": tau_f, "tau_g": tau_g,
                  "xi": xi, "hist": hist}))
