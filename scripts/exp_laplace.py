"""Exploration for the physics pins (tests/test_gpu_physics.py): droplet
pressure jump vs 2 sigma / R, and the resolved tanh profile, printed for
several run lengths.  GPU only; prints one line per case."""

import sys
import os

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1405_6162_b200 as lk  # noqa: E402
from paper_1405_6162_b200.lattice import FieldDescriptor, field_create  # noqa: E402


def state(shape, phi, model):
    desc = FieldDescriptor.create(19, shape.nsites)
    f, g = field_create(desc), field_create(desc)
    for i in range(19):
        f.component(i)[:] = model.wv[i]
        g.component(i)[:] = model.wv[i] * phi.ravel()
    return f, g


def moments(f, g, shape):
    n, P = shape.nsites, f.descriptor.padded_sites
    F = f.data.reshape(19, P)[:, :n]
    G = g.data.reshape(19, P)[:, :n]
    rho = F.sum(0)
    u = (lk.D3Q19Model().cvf.T @ F) / rho
    return rho, u, G.sum(0)


def droplet(R, steps_list, L=64, shift=True, fe=None):
    fe = fe or lk.FreeEnergy()
    sigma = np.sqrt(-8 * fe.kappa * fe.A ** 3 / (9 * fe.B ** 2))
    xi = np.sqrt(-2 * fe.kappa / fe.A)
    shape = lk.LatticeShape(L, L, L)
    x = np.indices((L, L, L)) - (L / 2 - 0.5)
    r = np.sqrt((x ** 2).sum(0))
    fpp = fe.A + 3 * fe.B * (-fe.A / fe.B)
    phis = np.sqrt(-fe.A / fe.B)
    d = (sigma / R / phis) / fpp if shift else 0.0
    phi0 = -phis * np.tanh((r - R) / xi) + d
    model = lk.D3Q19Model()
    f0, g0 = state(shape, phi0, model)
    done = 0
    with lk.BinaryFluid(shape, model=model, free_energy=fe, physics="binary") as sim:
        sim.load(f0, g0)
        for st in steps_list:
            sim.run(st - done)
            done = st
            f1, g1 = sim.fields()
            phi, mu = sim.order_parameter()
            rho, u, ph = moments(f1, g1, shape)
            rho3, ph3 = rho.reshape(L, L, L), ph.reshape(L, L, L)
            mu3 = mu.transpose(2, 1, 0)
            # radius from the phi = (phi_in + phi_out)/2 crossing along the radial profile
            rb = np.round(r).astype(int)
            prof = np.bincount(rb.ravel(), ph3.ravel()) / np.bincount(rb.ravel())
            pin, pout = float(ph3[r < 3].mean()), float(ph3[r > L / 2 - 2].mean())
            mid = 0.5 * (pin + pout)
            k = int(np.argmax(prof < mid))
            Rz = (k - 1) + (prof[k - 1] - mid) / (prof[k - 1] - prof[k])
            Pc = ph3 * mu3 - (fe.A / 2 * ph3 ** 2 + fe.B / 4 * ph3 ** 4)
            inside, outside = r < Rz - 4 * xi, r > Rz + 6 * xi
            dPc = float(Pc[inside].mean() - Pc[outside].mean())
            dPr = float((rho3[inside].mean() - rho3[outside].mean()) / 3)
            mu_in, mu_out = float(mu3[inside].mean()), float(mu3[outside].mean())
            print(f"R0={R:5.1f} steps={st:6d} Rz={Rz:6.3f} phi_in={pin:.5f} phi_out={pout:.5f} "
                  f"mu_in={mu_in:.3e} mu_out={mu_out:.3e} sigma/R={sigma / Rz:.3e} "
                  f"dPchem={dPc:.4e} dPrho={dPr:.3e} 2sig/R={2 * sigma / Rz:.4e} "
                  f"ratio={(dPc + dPr) / (2 * sigma / Rz):.4f} max|u|={np.abs(u).max():.2e}",
                  flush=True)


def tanh_profile(xi_case, steps_list, width=1.0):
    A, B, kappa = xi_case
    fe = lk.FreeEnergy(A=A, B=B, kappa=kappa)
    xi = np.sqrt(-2 * kappa / A)
    nz = 192 if xi <= 8 else 384
    shape = lk.LatticeShape(2, 2, nz)
    z = np.arange(nz)
    prof0 = np.tanh((z - nz / 4 + 0.5) / (width * xi)) * np.tanh((3 * nz / 4 - 0.5 - z) / (width * xi))
    phi0 = np.broadcast_to(prof0, (2, 2, nz)).copy()
    model = lk.D3Q19Model()
    f0, g0 = state(shape, phi0, model)
    done = 0
    with lk.BinaryFluid(shape, model=model, free_energy=fe, physics="binary") as sim:
        sim.load(f0, g0)
        for st in steps_list:
            sim.run(st - done)
            done = st
            f1, g1 = sim.fields()
            phi, mu = sim.order_parameter()
            _, u, ph = moments(f1, g1, shape)
            pz = ph.reshape(2, 2, nz).mean(axis=(0, 1))
            cross = [k + pz[k] / (pz[k] - pz[(k + 1) % nz]) for k in range(nz)
                     if pz[k] * pz[(k + 1) % nz] < 0]
            z1, z2 = sorted(cross)[:2]
            model_p = np.tanh((z - z1) / xi) * np.tanh((z2 - z) / xi)
            print(f"xi={xi:.1f} w={width} steps={st:7d} max|phi-tanh|={np.abs(pz - model_p).max():.3e} "
                  f"mu spread={np.ptp(mu):.3e} max|u|={np.abs(u).max():.2e} z={z1:.3f},{z2:.3f}",
                  flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "tanh"):
        tanh_profile((-0.002, 0.002, 0.064), [5000, 20000, 50000, 100000])
        tanh_profile((-0.001, 0.001, 0.128), [5000, 20000, 50000])
    if what in ("all", "laplace"):
        for R in (8.0, 10.0, 12.0, 16.0):
            droplet(R, [2000, 6000, 20000])
        droplet(12.0, [2000, 6000, 20000], shift=False)
