"""The oracle, pinned against the reference's own golden vectors (CPU only).

tests/golden/* were produced by the reference (tests/golden/make_golden.py);
here we prove the C restatement (oracle/lb_oracle.c) and the pure-Python
restatement reproduce them bitwise, then pin the builder-defined full-step
extension with known-answer tests.
"""

import hashlib

import numpy as np
import pytest

from oracle import oracle as orc


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


class TestCollisionPinnedToReference:
    def test_initial_state_generator_matches_reference(self, golden):
        meta, _ = golden
        for case in meta["collision"]:
            nx, ny, nz = case["shape"]
            f, g = orc.random_binary_state(nx * ny * nz, case["padded"], case["seed"])
            assert sha(f) == case["in_f"] and sha(g) == case["in_g"], case["shape"]

    def test_c_oracle_bitwise_vs_reference(self, golden):
        meta, _ = golden
        for case in meta["collision"]:
            nx, ny, nz = case["shape"]
            n, p = nx * ny * nz, case["padded"]
            f, g = orc.random_binary_state(n, p, case["seed"])
            bad = orc.collide(f, g, p, n, tau_f=case["tau_f"], tau_g=case["tau_g"],
                              steps=case["steps"])
            assert bad == -1
            assert sha(f) == case["out_f"], case
            assert sha(g) == case["out_g"], case

    def test_parallel_driver_bitwise(self, golden):
        meta, _ = golden
        case = [c for c in meta["collision"] if c["shape"] == [32, 32, 32]][0]
        n, p = 32 ** 3, case["padded"]
        f, g = orc.random_binary_state(n, p, case["seed"])
        orc.collide(f, g, p, n, tau_f=case["tau_f"], tau_g=case["tau_g"],
                    steps=case["steps"], threads=4)
        assert sha(f) == case["out_f"] and sha(g) == case["out_g"]

    def test_pure_python_restatement_bitwise(self, golden):
        _, small = golden
        for key in [k for k in small if k.startswith("coll_") and k.endswith("_in_f")]:
            stem = key[:-5]
            f, g = small[stem + "_in_f"].copy(), small[stem + "_in_g"].copy()
            dims = [int(v) for v in stem.split("_")[1].split("x")]
            n = dims[0] * dims[1] * dims[2]
            p = f.size // 19
            meta = [c for c in golden[0]["collision"] if c["shape"] == dims][0]
            for _ in range(meta["steps"]):
                orc.collide_scalar(f, g, p, n, tau_f=meta["tau_f"], tau_g=meta["tau_g"])
            assert np.array_equal(f.view(np.uint64), small[stem + "_out_f"].view(np.uint64))
            assert np.array_equal(g.view(np.uint64), small[stem + "_out_g"].view(np.uint64))

    def test_equilibrium_fixed_point_vector(self, golden):
        _, small = golden
        f, g = small["eqstate_in_f"].copy(), small["eqstate_in_g"].copy()
        p = f.size // 19
        orc.collide(f, g, p, 64)
        assert np.array_equal(f, small["eqstate_out_f"])
        assert np.array_equal(g, small["eqstate_out_g"])

    def test_singular_state_reported(self):
        f = np.zeros(19 * 16)
        g = np.zeros(19 * 16)
        assert orc.collide(f, g, 16, 8) == 0

    def test_padding_skipped(self, golden):
        _, small = golden
        f = small["coll_3x3x3_s6_in_f"].copy()
        g = small["coll_3x3x3_s6_in_g"].copy()
        assert orc.collide(f, g, 32, 27) == -1
        assert not f.reshape(19, 32)[:, 27:].any()


class TestScaleAndMaskPinned:
    def test_scale(self, golden):
        _, small = golden
        a = small["scale_5x4x3_in"].copy()
        orc.scale(a, a.size // 3, 0.37)
        assert np.array_equal(a, small["scale_5x4x3_out"])

    def test_masked_copy(self, golden):
        _, small = golden
        k = 0
        while f"mask{k}_flags" in small:
            ncomp, nsites, padded = (int(v) for v in small[f"mask{k}_meta"])
            dst = small[f"mask{k}_init"].copy()
            orc.masked_copy(dst, small[f"mask{k}_host"], ncomp, padded, small[f"mask{k}_flags"])
            assert np.array_equal(dst, small[f"mask{k}_out"])
            k += 1
        assert k == 12


# ------------------------------------------------------------ full-step extension

SHAPE = (6, 5, 4)


def _state(shape=SHAPE, seed=7):
    n = shape[0] * shape[1] * shape[2]
    p = -(-n // 16) * 16
    f, g = orc.random_binary_state(n, p, seed)
    return f, g, n, p


class TestStreaming:
    def test_single_population_moves_by_c(self):
        nx, ny, nz = 5, 4, 3
        n = nx * ny * nz
        p = 64
        for i in range(19):
            f = np.zeros(19 * p)
            x, y, z = 2, 1, 1
            f[i * p + (x * ny + y) * nz + z] = 1.0
            out = np.zeros_like(f)
            orc.lib().orc_stream(orc._p(f), orc._p(out), 19, p, nx, ny, nz)
            cx, cy, cz = orc.CV[i]
            dst = (((x + cx) % nx) * ny + (y + cy) % ny) * nz + (z + cz) % nz
            assert out[i * p + dst] == 1.0 and out.sum() == 1.0

    def test_stream_matches_numpy_roll(self):
        f, g, n, p = _state()
        out = np.zeros_like(f)
        orc.lib().orc_stream(orc._p(f), orc._p(out), 19, p, *SHAPE)
        assert np.array_equal(out, orc.stream_numpy(f, SHAPE, p))

    def test_stream_then_inverse_is_identity(self):
        f, g, n, p = _state()
        fwd = orc.stream_numpy(f, SHAPE, p)
        back = fwd.copy()
        nx, ny, nz = SHAPE
        for i in range(19):
            comp = fwd[i * p:i * p + n].reshape(nx, ny, nz)
            back[i * p:i * p + n] = np.roll(comp, tuple(-orc.CV[i]), (0, 1, 2)).ravel()
        assert np.array_equal(back, f)


class TestStencils:
    def test_laplacian_exact_on_quadratic(self):
        nx, ny, nz = 8, 8, 8
        x, y, z = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
        # periodic quadratic is impossible; check interior sites of a quadratic
        phi = (0.5 * x * x + 0.25 * y * y - 0.125 * z * z).astype(np.float64).ravel()
        mu = np.zeros_like(phi)
        orc.lib().orc_mu(orc._p(phi), orc._p(mu), nx, ny, nz, 0.0, 0.0, -1.0)
        lap = mu.reshape(nx, ny, nz)  # kappa = -1 -> mu = +lap
        assert np.allclose(lap[1:-1, 1:-1, 1:-1], 2 * (0.5 + 0.25 - 0.125), rtol=0, atol=1e-12)

    def test_mu_bulk_term(self):
        phi = np.full(4 * 4 * 4, 0.3)
        mu = np.zeros_like(phi)
        orc.lib().orc_mu(orc._p(phi), orc._p(mu), 4, 4, 4, -0.0625, 0.0625, 0.04)
        assert np.allclose(mu, -0.0625 * 0.3 + 0.0625 * 0.027, rtol=1e-15)


class TestFullStep:
    @pytest.mark.parametrize("physics", [0, 1, 2])
    def test_c_and_numpy_restatements_agree_bitwise(self, physics):
        f, g, n, p = _state()
        prm = orc.fluid_params(tau_f=0.8, tau_g=1.1, physics=physics)
        fc, gc, phic, muc = orc.fluid_step(f, g, SHAPE, p, prm, steps=1)
        fn, gn, phin, mun = orc.fluid_step_numpy(f, g, SHAPE, p, prm)
        assert np.array_equal(fc.view(np.uint64), fn.view(np.uint64))
        assert np.array_equal(gc.view(np.uint64), gn.view(np.uint64))
        assert np.array_equal(phic, phin)
        if physics:
            assert np.array_equal(muc, mun)

    def test_passive_limit_is_reference_collision_after_streaming(self, golden):
        # physics 0 == stream then the pinned reference collision, bitwise
        f, g, n, p = _state()
        prm = orc.fluid_params(tau_f=0.8, tau_g=1.3, physics=0)
        fo, go, _, _ = orc.fluid_step(f, g, SHAPE, p, prm, steps=1)
        fs, gs = orc.stream_numpy(f, SHAPE, p), orc.stream_numpy(g, SHAPE, p)
        orc.collide(fs, gs, p, n, tau_f=0.8, tau_g=1.3)
        assert np.array_equal(fo, fs) and np.array_equal(go, gs)

    def test_global_mass_and_phi_conserved(self):
        f, g, n, p = _state((8, 8, 8), 3)
        prm = orc.fluid_params(tau_f=0.9, tau_g=1.0, physics=1)
        fo, go, _, _ = orc.fluid_step(f, g, (8, 8, 8), p, prm, steps=5)
        assert abs(fo.sum() - f.sum()) <= 1e-12 * f.sum()
        assert abs(go.sum() - g.sum()) <= 1e-12 * abs(g.sum())

    def test_momentum_changes_by_total_force(self):
        shape = (8, 6, 4)
        f, g, n, p = _state(shape, 9)
        prm = orc.fluid_params(tau_f=0.9, tau_g=1.0, physics=1)
        fo, go, phi, mu = orc.fluid_step(f, g, shape, p, prm, steps=1)
        cv = orc.CV.astype(float)
        fs = orc.stream_numpy(f, shape, p).reshape(19, p)[:, :n]
        F = np.stack([c.ravel() for c in orc.potential_force_numpy(phi.reshape(shape),
                                                                  mu.reshape(shape))])
        before = cv.T @ fs
        after = cv.T @ fo.reshape(19, p)[:, :n]
        assert np.allclose(after - before, F, rtol=0, atol=1e-14)

    def test_uniform_equilibrium_is_fixed_point(self):
        # uniform phi -> mu uniform -> no force; g_eq includes lam*(gamma mu - phi cs2)
        shape = (4, 4, 4)
        n, p = 64, 64
        prm = orc.fluid_params(tau_f=0.8, tau_g=1.2, physics=1)
        rho, u, phi0 = 1.0, np.array([0.02, -0.01, 0.03]), 0.3
        cv = orc.CV.astype(float)
        cs2 = orc.CS2
        mu0 = prm.A * phi0 + prm.B * phi0 ** 3
        lam = orc.lam_weights()
        f = np.zeros(19 * p)
        g = np.zeros(19 * p)
        for i in range(19):
            ud = cv[i] @ u
            br = 1 + ud / cs2 + ud * ud / (2 * cs2 * cs2) - (u @ u) / (2 * cs2)
            f[i * p:(i + 1) * p] = orc.WV[i] * rho * br
            g[i * p:(i + 1) * p] = orc.WV[i] * phi0 * br + lam[i] * (prm.gamma * mu0 - phi0 * cs2)
        fo, go, _, _ = orc.fluid_step(f, g, shape, p, prm, steps=3)
        assert np.max(np.abs(fo - f)) < 1e-14 and np.max(np.abs(go - g)) < 1e-14

    def test_flat_interface_near_stationary(self):
        # phi = tanh(z/xi) profile (xi = sqrt(-2 kappa/A) ~ 1.13) is the
        # continuum stationary interface.  The lattice relaxes it to its
        # discrete profile (<0.1 from tanh) and then holds it: the interfaces
        # do not move and the bulk stays at phi* = +-1.
        nx, ny, nz = 4, 4, 32
        n = p = nx * ny * nz
        prm = orc.fluid_params(tau_f=1.0, tau_g=1.0, physics=1)
        xi = np.sqrt(-2 * prm.kappa / prm.A)
        z = np.arange(nz)
        prof = np.tanh((z - nz / 4 + 0.5) / xi) * -np.tanh((z - 3 * nz / 4 + 0.5) / xi)
        phi = np.broadcast_to(prof, (nx, ny, nz)).ravel()
        lam = orc.lam_weights()
        f = np.zeros(19 * p)
        g = np.zeros(19 * p)
        for i in range(19):
            f[i * p:(i + 1) * p] = orc.WV[i]
            g[i * p:(i + 1) * p] = orc.WV[i] * phi + lam[i] * (0.0 - phi * orc.CS2)
        f, g, phi1, _ = orc.fluid_step(f, g, (nx, ny, nz), p, prm, steps=100)
        f, g, phi2, _ = orc.fluid_step(f, g, (nx, ny, nz), p, prm, steps=100)
        assert np.max(np.abs(phi1 - phi)) < 0.1
        assert np.max(np.abs(phi2 - phi1)) < 5e-3
        assert np.array_equal(np.sign(phi2), np.sign(phi))
        assert np.min(np.abs(phi2.reshape(nx, ny, nz)[:, :, [0, 15, 16, 31]])) > 0.99


def _double_interface(shape, prm):
    """Periodic double flat interface at rest: f_i = w_i, g_i = w_i phi(z),
    phi = tanh((z - nz/4 + 1/2)/xi) tanh((3nz/4 - 1/2 - z)/xi)."""
    nx, ny, nz = shape
    n = nx * ny * nz
    p = -(-n // 16) * 16
    xi = np.sqrt(-2 * prm.kappa / prm.A)
    z = np.arange(nz)
    prof = np.tanh((z - nz / 4 + 0.5) / xi) * np.tanh((3 * nz / 4 - 0.5 - z) / xi)
    phi = np.broadcast_to(prof, shape).ravel()
    f = np.zeros(19 * p)
    g = np.zeros(19 * p)
    for i in range(19):
        f[i * p:i * p + n] = orc.WV[i]
        g[i * p:i * p + n] = orc.WV[i] * phi
    return f, g, n, p


def _max_u(f, n, p):
    F = f.reshape(19, p)[:, :n]
    return float(np.max(np.abs((orc.CV.astype(float).T @ F) / F.sum(0))))


class TestStressForm:
    """physics 2: the same fluid with the force as the divergence of the chemical
    pressure tensor, F = -div P (continuum-equal to -phi grad mu).  A discrete
    divergence telescopes, so the lattice momentum is conserved to rounding, and
    the flat interface the -phi grad mu form destabilises stays put."""

    def test_momentum_conserved(self):
        shape = (8, 6, 4)
        f, g, n, p = _state(shape, 9)
        prm = orc.fluid_params(tau_f=0.9, tau_g=1.0, physics=2)
        cv = orc.CV.astype(float)
        before = cv.T @ f.reshape(19, p)[:, :n]
        fo, go, _, _ = orc.fluid_step(f, g, shape, p, prm, steps=3)
        after = cv.T @ fo.reshape(19, p)[:, :n]
        assert np.allclose(after.sum(1), before.sum(1), rtol=0, atol=1e-13)
        assert abs(fo.sum() - f.sum()) <= 1e-12 * f.sum()
        assert abs(go.sum() - g.sum()) <= 1e-12 * abs(g.sum())

    def test_force_equals_phi_grad_mu_on_smooth_field(self):
        # div P = phi grad mu in the continuum: on a smooth periodic profile the
        # two discrete forces agree to the stencils' O(h^2)
        nx, ny, nz = 4, 4, 64
        z = np.arange(nz)
        p3 = np.broadcast_to(0.8 * np.sin(2 * np.pi * z / nz), (nx, ny, nz)).copy()
        prm = orc.fluid_params(physics=2, A=-0.0625, B=0.0625, kappa=0.04)
        mu3 = orc.mu_numpy(p3, [np.roll(p3, s, a) for a in range(3) for s in (-1, 1)], prm)
        F = orc.stress_force_numpy(p3, mu3, prm)
        Fpot = -(p3 * ((np.roll(mu3, -1, 2) - np.roll(mu3, 1, 2)) * 0.5))
        assert np.max(np.abs(F[2] - Fpot)) < 0.05 * np.max(np.abs(Fpot))
        assert np.max(np.abs(F[0])) < 1e-15 and np.max(np.abs(F[1])) < 1e-15
        assert abs(F[2].sum()) < 1e-14

    def test_flat_interface_both_forms_stable(self):
        # Ludwig-scale constants (A = -B = 0.0625, kappa = 0.04, xi = 1.13):
        # the filtered potential form (physics 1) relaxes a flat double
        # interface to rest -- |u| decays exponentially, ~3x per 2000 steps --
        # while the stress divergence (physics 2) holds it with a spurious
        # velocity ~1e-4 (its discrete F is not zero where mu is uniform).
        shape = (2, 2, 64)
        res = {}
        for physics in (1, 2):
            prm = orc.fluid_params(tau_f=1.0, tau_g=1.0, physics=physics, A=-0.0625, B=0.0625,
                                   kappa=0.04)
            f, g, n, p = _double_interface(shape, prm)
            f, g, _, _ = orc.fluid_step(f, g, shape, p, prm, steps=1500)
            u1 = _max_u(f, n, p)
            f, g, phi, _ = orc.fluid_step(f, g, shape, p, prm, steps=1500)
            res[physics] = (u1, _max_u(f, n, p), float(np.max(phi)))
        assert res[1][1] < 1e-5 and res[1][1] < 0.5 * res[1][0]   # decaying to rest
        assert res[2][1] < 5e-4 and res[2][1] < 2 * res[2][0] + 1e-5
        assert res[1][2] > 0.99 and res[2][2] > 0.99


class TestPotentialForm:
    """physics 1: why -phi grad mu is filtered along its own axis."""

    def test_staggered_momentum_mode_is_undamped(self):
        # j_z with wavenumber pi along z flips sign under one stream+collide
        # step and keeps its magnitude, for any tau: momentum is a collision
        # invariant and the moving populations all change sublattice.  This is
        # the mode the unfiltered potential force pumped.
        shape = (1, 1, 8)
        n = p = 8
        prm = orc.fluid_params(tau_f=0.8, tau_g=1.0, physics=0)
        cv = orc.CV.astype(float)
        uz = 1e-3 * (-1.0) ** np.arange(8)
        f = np.zeros(19 * p)
        g = np.zeros(19 * p)
        for i in range(19):
            ud = cv[i, 2] * uz
            f[i * p:(i + 1) * p] = orc.WV[i] * (1 + 3 * ud + 4.5 * ud * ud - 1.5 * uz * uz)
            g[i * p:(i + 1) * p] = orc.WV[i] * 0.3
        jz0 = cv[:, 2] @ f.reshape(19, p)
        fo, _, _, _ = orc.fluid_step(f, g, shape, p, prm, steps=1)
        jz1 = cv[:, 2] @ fo.reshape(19, p)
        assert np.allclose(jz1, -jz0, rtol=0, atol=1e-15)

    def test_unfiltered_force_would_project_on_it(self):
        # the raw -phi grad mu of a tanh interface has a nonzero (-1)^z
        # component; the filtered force has none
        nz = 32
        z = np.arange(nz)
        p3 = np.broadcast_to(np.tanh((z - 8.3) / 1.13) * np.tanh((23.7 - z) / 1.13),
                             (1, 1, nz)).copy()
        p3 += 1e-3 * (-1.0) ** z * np.exp(-((z - 8.3) / 3) ** 2)  # checkerboard at one interface
        prm = orc.fluid_params(physics=1)
        mu3 = orc.mu_numpy(p3, [np.roll(p3, s, a) for a in range(3) for s in (-1, 1)], prm)
        h = -(p3 * ((np.roll(mu3, -1, 2) - np.roll(mu3, 1, 2)) * 0.5))
        F = orc.potential_force_numpy(p3, mu3)[2]
        stag = (-1.0) ** z
        assert abs(float((h * stag).sum())) > 1e-5
        assert abs(float((F * stag).sum())) < 1e-17

    def test_zero_where_mu_uniform(self):
        rng = np.random.default_rng(3)
        p3 = rng.uniform(-1, 1, (4, 5, 6))
        mu3 = np.full_like(p3, 0.123)
        for comp in orc.potential_force_numpy(p3, mu3):
            assert np.all(comp == 0.0)


def test_fluid_stepper_equals_fluid_step():
    # bench.py's CPU timing path (preallocated buffers) computes the same steps
    shape = (6, 5, 4)
    f, g, n, p = _state(shape, 3)
    prm = orc.fluid_params(tau_f=0.9, tau_g=1.1, physics=1)
    ref_f, ref_g, _, _ = orc.fluid_step(f, g, shape, p, prm, steps=3)
    st = orc.FluidStepper(shape, p, prm)
    st.load(f, g)
    st.run(1)
    st.run(2)
    sf, sg = st.state()
    assert np.array_equal(sf, ref_f) and np.array_equal(sg, ref_g)


# ------------------------------------------------------------ properties (hypothesis)

from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

_dims = st.tuples(st.integers(1, 6), st.integers(1, 6), st.integers(1, 6))


@settings(max_examples=25, deadline=None)
@given(shape=_dims, seed=st.integers(0, 2 ** 31 - 1))
def test_property_stream_c_equals_numpy_and_inverts(shape, seed):
    n = shape[0] * shape[1] * shape[2]
    p = -(-n // 16) * 16
    rng = np.random.default_rng(seed)
    f = np.zeros(19 * p)
    f.reshape(19, p)[:, :n] = rng.random((19, n))
    out = np.zeros_like(f)
    orc.lib().orc_stream(orc._p(f), orc._p(out), 19, p, *shape)
    assert np.array_equal(out, orc.stream_numpy(f, shape, p))
    # pulling every component by -c_i undoes the stream
    back = np.zeros_like(f)
    o3 = out.reshape(19, p)[:, :n].reshape(19, *shape)
    for i in range(19):
        back.reshape(19, p)[i, :n] = np.roll(o3[i], tuple(-c for c in orc.CV[i]),
                                             axis=(0, 1, 2)).ravel()
    assert np.array_equal(back, f)


@settings(max_examples=25, deadline=None)
@given(shape=_dims, seed=st.integers(0, 2 ** 31 - 1))
def test_property_stress_force_sums_to_zero(shape, seed):
    # a discrete divergence telescopes on any periodic lattice
    rng = np.random.default_rng(seed)
    p3 = rng.uniform(-1, 1, shape)
    prm = orc.fluid_params(physics=2)
    mu3 = orc.mu_numpy(p3, [np.roll(p3, s, a) for a in range(3) for s in (-1, 1)], prm)
    F = orc.stress_force_numpy(p3, mu3, prm)
    scale = max(1.0, float(max(np.abs(f).max() for f in F)))
    for comp in F:
        assert abs(comp.sum()) <= 1e-13 * scale * comp.size


@settings(max_examples=25, deadline=None)
@given(shape=st.tuples(st.integers(1, 4), st.integers(1, 4), st.integers(1, 4)),
       seed=st.integers(0, 2 ** 31 - 1))
def test_property_potential_force_filtered(shape, seed):
    # on any periodic lattice with even extents: no component on the
    # wavenumber-pi mode of its own axis, and the filter keeps sum_x F
    shape = tuple(2 * d for d in shape)
    rng = np.random.default_rng(seed)
    p3, mu3 = rng.uniform(-1, 1, shape), rng.uniform(-1, 1, shape)
    F = orc.potential_force_numpy(p3, mu3)
    for a in range(3):
        h = -(p3 * ((np.roll(mu3, -1, a) - np.roll(mu3, 1, a)) * 0.5))
        idx = np.indices(shape)[a]
        assert abs(float((F[a] * (-1.0) ** idx).sum())) <= 1e-14 * F[a].size
        assert abs(float(F[a].sum() - h.sum())) <= 1e-14 * F[a].size


@settings(max_examples=15, deadline=None)
@given(shape=_dims, seed=st.integers(0, 2 ** 31 - 1), physics=st.sampled_from([0, 1, 2]),
       tau_f=st.sampled_from([0.6, 1.0, 1.7]), tau_g=st.sampled_from([0.7, 1.0]))
def test_property_c_and_numpy_full_step_bitwise(shape, seed, physics, tau_f, tau_g):
    n = shape[0] * shape[1] * shape[2]
    p = -(-n // 16) * 16
    f, g = orc.random_binary_state(n, p, seed)
    prm = orc.fluid_params(tau_f=tau_f, tau_g=tau_g, physics=physics)
    fc, gc, _, _ = orc.fluid_step(f, g, shape, p, prm, steps=1)
    fn, gn, _, _ = orc.fluid_step_numpy(f, g, shape, p, prm)
    assert np.array_equal(fc.view(np.uint64), fn.view(np.uint64))
    assert np.array_equal(gc.view(np.uint64), gn.view(np.uint64))
