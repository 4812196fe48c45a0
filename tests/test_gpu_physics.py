"""Physics pins of the builder-defined free-energy extension.

The reference has no chemical potential, force or streaming (reference
SPEC.md:393-405, pkg/README.md:34-35), so the GPU-vs-oracle parity tests can
only show that the CUDA path computes the oracle's formulas.  These tests tie
the formulas to the published physics of the symmetric binary free energy
f = A/2 phi^2 + B/4 phi^4 + kappa/2 |grad phi|^2 (Ludwig's binary fluid,
Kendon et al. 2001; Desplat, Pagonabarraga & Bladon 2001):

* a flat interface relaxes to rest: the spurious velocity decays below 1e-6
  (the filtered potential force is exactly zero where mu is uniform);
* the interface profile is phi* tanh(z / xi), phi* = sqrt(-A/B),
  xi = sqrt(-2 kappa / A) (to 1e-3 on a resolved interface; at the default
  xi = 1.13 the lattice profile is the exact discrete equilibrium, mu uniform);
* Laplace's law dP = 2 sigma / R on 3-D droplets with
  sigma = sqrt(-8 kappa A^3 / (9 B^2)).
All run in EXACT mode (the benchmarked arithmetic).
"""

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def lk():
    import paper_1405_6162_b200 as lk

    return lk


def _state(lk, shape, phi, model):
    """f_i = w_i (rho = 1, u = 0), g_i = w_i phi (host order (x, y, z))."""
    from paper_1405_6162_b200.lattice import FieldDescriptor, field_create

    desc = FieldDescriptor.create(19, shape.nsites)
    f, g = field_create(desc), field_create(desc)
    for i in range(19):
        f.component(i)[:] = model.wv[i]
        g.component(i)[:] = model.wv[i] * phi.ravel()
    return f, g


def _moments(lk, f, g, shape):
    n, P = shape.nsites, f.descriptor.padded_sites
    F = f.data.reshape(19, P)[:, :n]
    G = g.data.reshape(19, P)[:, :n]
    rho = F.sum(0)
    u = (lk.D3Q19Model().cvf.T @ F) / rho
    return rho, u, G.sum(0)


def _double_interface(nx, ny, nz, xi, width=1.0):
    z = np.arange(nz)
    prof = np.tanh((z - nz / 4 + 0.5) / (width * xi)) * np.tanh((3 * nz / 4 - 0.5 - z) /
                                                                  (width * xi))
    return np.broadcast_to(prof, (nx, ny, nz)).copy()


def _run(lk, shape, phi0, fe, steps, physics="binary", tau=1.0):
    model = lk.D3Q19Model(tau_f=tau, tau_g=tau)
    f0, g0 = _state(lk, shape, phi0, model)
    with lk.BinaryFluid(shape, model=model, free_energy=fe, physics=physics) as sim:
        sim.load(f0, g0)
        sim.run(steps)
        f1, g1 = sim.fields()
        phi, mu = sim.order_parameter()
    return f1, g1, phi, mu


class TestFlatInterface:
    def test_relaxes_to_rest(self, lk):
        # Ludwig's constants (A = -B = 0.0625, kappa = 0.04, xi = 1.13), a
        # periodic double interface started from the continuum tanh: after
        # 10^4 steps the spurious velocity is below 1e-6 and the bulk at phi*.
        fe = lk.FreeEnergy()
        shape = lk.LatticeShape(8, 8, 64)
        xi = np.sqrt(-2 * fe.kappa / fe.A)
        f1, g1, phi, mu = _run(lk, shape, _double_interface(8, 8, 64, xi), fe, 10000)
        rho, u, ph = _moments(lk, f1, g1, shape)
        umax = float(np.abs(u).max())
        print(f"flat interface, 10^4 steps: max|u| = {umax:.3e}")
        assert umax <= 1e-6
        assert 0.99 < ph.max() < 1.01 and -1.01 < ph.min() < -0.99
        # towards equilibrium: mu uniform (the discrete Euler-Lagrange
        # condition); the spread decays diffusively (1.1e-6 at 10^4 steps)
        spread = float(np.abs(mu - mu.mean()).max())
        print(f"flat interface, 10^4 steps: max|mu - <mu>| = {spread:.3e}")
        assert spread < 5e-6

    def test_stress_form_spurious_velocity(self, lk):
        # the divergence form holds the interface too, but its discrete force
        # is not zero where mu is uniform: spurious currents ~1e-4 (why the
        # potential form is the default)
        fe = lk.FreeEnergy()
        shape = lk.LatticeShape(8, 8, 64)
        xi = np.sqrt(-2 * fe.kappa / fe.A)
        f1, g1, _, _ = _run(lk, shape, _double_interface(8, 8, 64, xi), fe, 4000,
                            physics="binary-stress")
        _, u, ph = _moments(lk, f1, g1, shape)
        umax = float(np.abs(u).max())
        print(f"stress form, 4000 steps: max|u| = {umax:.3e}")
        assert 1e-6 < umax < 1e-3 and ph.max() > 0.99

    def test_sharp_step_relaxes(self, lk):
        # from a sharp step (phi = +-1) the interface forms, and the flow the
        # initial force kicks up decays (the unfiltered force grew it to 0.25)
        fe = lk.FreeEnergy()
        shape = lk.LatticeShape(4, 4, 64)
        z = np.arange(64)
        step = np.where((z >= 16) & (z < 48), 1.0, -1.0)
        phi0 = np.broadcast_to(step, (4, 4, 64)).copy()
        f1, g1, _, _ = _run(lk, shape, phi0, fe, 20000)
        _, u, ph = _moments(lk, f1, g1, shape)
        assert float(np.abs(u).max()) < 1e-8 and ph.max() > 0.99

    def test_discrete_profile_is_equilibrium(self, lk):
        # at xi = 1.13 the lattice resolves the interface with ~2 sites: the
        # steady profile is the discrete equilibrium (A phi + B phi^3 -
        # kappa lap phi = const), which differs from the continuum tanh by
        # up to ~0.07; check it against a Newton solve of that equation
        fe = lk.FreeEnergy()
        nz = 64
        shape = lk.LatticeShape(4, 4, nz)
        xi = np.sqrt(-2 * fe.kappa / fe.A)
        _, g1, phi, mu = _run(lk, shape, _double_interface(4, 4, nz, xi), fe, 10000)
        pz = phi.mean(axis=(1, 2))                     # (nz,)
        m0 = float(mu.mean())
        p = pz.copy()
        for _ in range(50):                            # Newton on the 1-D discrete equation
            lap = np.roll(p, 1) + np.roll(p, -1) - 2 * p
            r = fe.A * p + fe.B * p ** 3 - fe.kappa * lap - m0
            J = np.diag(fe.A + 3 * fe.B * p ** 2 + 2 * fe.kappa)
            for k in range(nz):
                J[k, (k + 1) % nz] -= fe.kappa
                J[k, (k - 1) % nz] -= fe.kappa
            p = p - np.linalg.solve(J, r)
        err = float(np.abs(pz - p).max())
        cont = _double_interface(1, 1, nz, xi)[0, 0]
        print(f"discrete profile: max|phi - Newton| = {err:.2e}, "
              f"max|phi - tanh| = {np.abs(pz - cont).max():.3f}")
        assert err < 5e-5


class TestInterfaceProfile:
    def test_tanh_profile_resolved_interface(self, lk):
        # xi = 8 (A = -B = -0.002, kappa = 0.064): the discrete equilibrium is
        # within 8.9e-4 of phi* tanh(z/xi) (1-D Newton solve of A phi + B phi^3
        # - kappa lap phi = 0).  Start from the continuum profile: the fluid
        # stays within 1e-3 of it while relaxing towards the discrete profile,
        # at rest (the relaxation of a mis-sized profile takes ~10^6 steps at
        # this mobility, so it is not a practical start)
        fe = lk.FreeEnergy(A=-0.002, B=0.002, kappa=0.064)
        xi = np.sqrt(-2 * fe.kappa / fe.A)
        nz = 192
        shape = lk.LatticeShape(2, 2, nz)
        f1, g1, phi, mu = _run(lk, shape, _double_interface(2, 2, nz, xi), fe, 50000)
        _, u, ph = _moments(lk, f1, g1, shape)
        pz = ph.reshape(2, 2, nz).mean(axis=(0, 1))
        z = np.arange(nz, dtype=float)
        cross = [k + pz[k] / (pz[k] - pz[(k + 1) % nz]) for k in range(nz)
                 if pz[k] * pz[(k + 1) % nz] < 0]
        z1, z2 = sorted(cross)[:2]
        model = np.tanh((z - z1) / xi) * np.tanh((z2 - z) / xi)
        err = float(np.abs(pz - model).max())
        umax = float(np.abs(u).max())
        print(f"tanh profile xi = {xi:.1f}: max|phi - phi* tanh| = {err:.2e}, interfaces "
              f"{z1:.2f} {z2:.2f}, max|u| = {umax:.1e}, mu spread {np.ptp(mu):.1e}")
        assert err <= 1e-3
        assert abs(z1 - (nz / 4 - 0.5)) < 1e-3 and abs(z2 - (3 * nz / 4 - 0.5)) < 1e-3
        assert umax < 1e-6


class TestLaplaceLaw:
    def test_droplet_pressure_jump(self, lk):
        # 3-D droplets of radius 8..16 in a 64^3 periodic box.  Each starts with
        # its bulk values shifted by mu0 / f''(phi*), mu0 = sigma / (R phi*) (the
        # Gibbs-Thomson shift; without it the droplet first evaporates into the
        # finite box).  After 6000 steps the pressure jump between the bulk
        # phases, P = rho cs2 + phi mu - (A/2 phi^2 + B/4 phi^4), is 2 sigma / R
        # with sigma = sqrt(-8 kappa A^3 / (9 B^2)), R the radius where phi
        # crosses the mean of the two bulk values
        fe = lk.FreeEnergy()
        sigma = np.sqrt(-8 * fe.kappa * fe.A ** 3 / (9 * fe.B ** 2))
        xi = np.sqrt(-2 * fe.kappa / fe.A)
        phis = np.sqrt(-fe.A / fe.B)
        fpp = fe.A + 3 * fe.B * phis ** 2
        L = 64
        shape = lk.LatticeShape(L, L, L)
        x = np.indices((L, L, L)) - (L / 2 - 0.5)
        r = np.sqrt((x ** 2).sum(0))
        rb = np.round(r).astype(int).ravel()
        cnt = np.bincount(rb)
        inv_r, dp, umax = [], [], []
        for R in (8.0, 10.0, 12.0, 16.0):
            phi0 = -phis * np.tanh((r - R) / xi) + sigma / (R * phis) / fpp
            f1, g1, phi, mu = _run(lk, shape, phi0, fe, 6000)
            rho, u, ph = _moments(lk, f1, g1, shape)
            rho3, ph3 = rho.reshape(L, L, L), ph.reshape(L, L, L)
            mu3 = mu.transpose(2, 1, 0)                # device (z, y, x) -> host (x, y, z)
            pin, pout = float(ph3[r < 3].mean()), float(ph3[r > L / 2 - 2].mean())
            mid = 0.5 * (pin + pout)
            with np.errstate(invalid="ignore"):  # radii no lattice point rounds to: NaN, skipped
                prof = np.bincount(rb, ph3.ravel())[:L // 2] / cnt[:L // 2]
            k = int(np.argmax(prof < mid))
            Rz = (k - 1) + (prof[k - 1] - mid) / (prof[k - 1] - prof[k])
            P = rho3 / 3 + ph3 * mu3 - (fe.A / 2 * ph3 ** 2 + fe.B / 4 * ph3 ** 4)
            inside, outside = r < Rz - 4 * xi, r > Rz + 6 * xi
            inv_r.append(1 / Rz)
            dp.append(float(P[inside].mean() - P[outside].mean()))
            umax.append(float(np.abs(u).max()))
        slope, icpt = np.polyfit(inv_r, dp, 1)
        print(f"Laplace: sigma fit {slope / 2:.5f} vs analytic {sigma:.5f} "
              f"({slope / 2 / sigma - 1:+.2%}), intercept {icpt:.1e}; "
              f"R = {[round(1 / v, 2) for v in inv_r]}, "
              f"dP / (2 sigma / R) = {[round(v / (2 * sigma * ir), 4) for v, ir in zip(dp, inv_r)]}, "
              f"max|u| = {[f'{v:.1e}' for v in umax]}")
        assert abs(slope / 2 / sigma - 1) <= 0.05
        for v, ir in zip(dp, inv_r):
            assert abs(v / (2 * sigma * ir) - 1) <= 0.05
        assert max(umax) < 1e-4
