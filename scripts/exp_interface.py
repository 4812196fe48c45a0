"""Physics check of the builder-defined full step on the GPU: a
periodic double flat interface relaxes to the analytic profile of the symmetric
free energy, phi(z) = phi* tanh(z / xi), phi* = sqrt(-A/B), xi = sqrt(-2 kappa / A).

Initial state: rho = 1, u = 0 (f_i = w_i), g_i = w_i phi0(z) with a sharp step
profile; after N steps the x,y-averaged phi(z) is compared with the two-interface
tanh profile centred where phi crosses zero, and the spurious velocity is read
from the f moments.  Prints one JSON line."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1405_6162_b200 as lk  # noqa: E402
from paper_1405_6162_b200.lattice import FieldDescriptor, field_create  # noqa: E402

nx, ny, nz = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "32x32x128").split("x"))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
mode = lk.MODE_EXACT if (len(sys.argv) > 3 and sys.argv[3] == "exact") else lk.MODE_FAST
# optional: A B kappa gamma tau_f tau_g
kv = dict(zip(["A", "B", "kappa", "gamma", "tau_f", "tau_g"], map(float, sys.argv[4:10])))
fe = lk.FreeEnergy(**{k: kv[k] for k in ("A", "B", "kappa", "gamma") if k in kv})
model = lk.D3Q19Model(tau_f=kv.get("tau_f", 1.0), tau_g=kv.get("tau_g", 1.0))
phis, xi = np.sqrt(-fe.A / fe.B), np.sqrt(-2 * fe.kappa / fe.A)
shape = lk.LatticeShape(nx, ny, nz)
desc = FieldDescriptor.create(19, shape.nsites)
f, g = field_create(desc), field_create(desc)
z = np.arange(nz)
prof0 = np.where((z >= nz // 4) & (z < 3 * nz // 4), 1.0, -1.0)          # sharp steps
phi0 = np.broadcast_to(prof0, (nx, ny, nz)).reshape(-1)                    # host order x,y,z
for i in range(19):
    f.component(i)[:] = model.wv[i]
    g.component(i)[:] = model.wv[i] * phi0
n, P = shape.nsites, desc.padded_sites
with lk.BinaryFluid(shape, model=model, free_energy=fe, mode=mode) as sim:
    sim.load(f, g)
    t0 = sim.totals()
    sim.run(steps)
    t1 = sim.totals()
    f1, g1 = sim.fields()
    phi_dev, mu_dev = sim.order_parameter()
F = f1.data.reshape(19, P)[:, :n]
G = g1.data.reshape(19, P)[:, :n]
rho = F.sum(0)
cv = model.cvf
j = np.stack([(cv[:, k][:, None] * F).sum(0) for k in range(3)])
umax = float(np.max(np.abs(j / rho)))
phi = G.sum(0).reshape(nx, ny, nz)
pz = phi.mean(axis=(0, 1))
spread = float(np.max(np.abs(phi - pz[None, None, :])))
# zero crossings (linear interpolation) -> interface positions
cross = []
for k in range(nz):
    a, b = pz[k], pz[(k + 1) % nz]
    if a * b < 0:
        cross.append(k + a / (a - b))
z1, z2 = sorted(cross)[:2]
zz = z.astype(float)
model_prof = phis * np.tanh((zz - z1) / xi) * np.tanh((z2 - zz) / xi)
model_prof = np.where((zz > z1) & (zz < z2), np.abs(model_prof), -np.abs(model_prof))
# away from the interfaces the double-tanh product saturates to +-phi*
err = float(np.max(np.abs(pz - model_prof)))
print(json.dumps({
    "shape": [nx, ny, nz], "steps": steps, "mode": "exact" if mode == lk.MODE_EXACT else "fast",
    "A": fe.A, "B": fe.B, "kappa": fe.kappa, "gamma": fe.gamma,
    "tau_f": model.tau_f, "tau_g": model.tau_g,
    "xi_analytic": xi, "phi_star": phis,
    "interfaces_at": [z1, z2], "max_abs_profile_error": err,
    "phi_min_max": [float(pz.min()), float(pz.max())],
    "xy_uniformity": spread, "max_spurious_velocity": umax,
    "mass_rel_drift": abs(t1[0] - t0[0]) / abs(t0[0]),
    "phi_abs_drift": abs(t1[4] - t0[4]),
    "finite": bool(np.isfinite(F).all() and np.isfinite(G).all())}))
