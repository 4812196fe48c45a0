"""GPU parity of the full timestep (collision + propagation + phi/mu stencils).

The engine (csrc/fluid.cu, BinaryFluid) against the C oracle
(oracle/lb_oracle.c orc_fluid_step, host order, independent indexing):
EXACT mode bitwise after N steps, FAST mode <= 1e-12 relative on f, g, rho,
phi (the north-star tolerance).  The passive limit must equal the reference
collision composed with streaming, which ties the extension to the pinned
reference arithmetic.  Slab decomposition is checked on one GPU by running
P virtual slabs through the C-ABI kernels with plane-copy halos, bitwise
equal to the single-slab run.
"""

import ctypes
import os

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def lk():
    import paper_1405_6162_b200 as lk

    return lk


def _state(lk, shape, seed):
    from paper_1405_6162_b200.kernels import random_binary_state

    return random_binary_state(lk.LatticeShape(*shape), np.random.default_rng(seed))


def _oracle(f0, g0, shape, steps, physics, tau_f=1.0, tau_g=1.0):
    from oracle import oracle as orc

    prm = orc.fluid_params(tau_f=tau_f, tau_g=tau_g, physics=physics)
    return orc.fluid_step(f0.data, g0.data, shape, f0.descriptor.padded_sites, prm, steps=steps,
                          threads=8)


SHAPES = [(16, 12, 10), (8, 8, 8), (32, 16, 6), (6, 10, 4)]


class TestFullStepParity:
    @pytest.mark.parametrize("shape", SHAPES)
    @pytest.mark.parametrize("physics", ["binary", "passive"])
    @pytest.mark.parametrize("graph", [True, False])
    def test_exact_bitwise(self, lk, shape, physics, graph):
        f0, g0 = _state(lk, shape, 7)
        model = lk.D3Q19Model(tau_f=0.8, tau_g=1.1)
        with lk.BinaryFluid(lk.LatticeShape(*shape), model=model, physics=physics,
                            use_graph=graph) as sim:
            sim.load(f0, g0)
            sim.run(4)
            f1, g1 = sim.fields()
            phi, mu = sim.order_parameter()
        of, og, ophi, omu = _oracle(f0, g0, shape, 4, 1 if physics == "binary" else 0, 0.8, 1.1)
        assert np.array_equal(f1.data.view(np.uint64), of.view(np.uint64))
        assert np.array_equal(g1.data.view(np.uint64), og.view(np.uint64))
        nx, ny, nz = shape
        # device (z, y, x) -> host (x, y, z)
        assert np.array_equal(phi.transpose(2, 1, 0).ravel(), ophi)
        if physics == "binary":
            assert np.array_equal(mu.transpose(2, 1, 0).ravel(), omu)

    @pytest.mark.parametrize("vvl", [1, 2])
    def test_vvl_bitwise(self, lk, vvl):
        shape = (16, 8, 8)
        f0, g0 = _state(lk, shape, 3)
        with lk.BinaryFluid(lk.LatticeShape(*shape), vvl=vvl) as sim:
            sim.load(f0, g0)
            sim.run(3)
            f1, g1 = sim.fields()
        of, og, _, _ = _oracle(f0, g0, shape, 3, 1)
        assert np.array_equal(f1.data, of) and np.array_equal(g1.data, og)

    def test_fast_within_1e12(self, lk):
        shape = (32, 32, 32)
        f0, g0 = _state(lk, shape, 11)
        model = lk.D3Q19Model(tau_f=0.9, tau_g=1.0)
        with lk.BinaryFluid(lk.LatticeShape(*shape), model=model, mode=lk.MODE_FAST) as sim:
            sim.load(f0, g0)
            sim.run(10)
            f1, g1 = sim.fields()
        of, og, _, _ = _oracle(f0, g0, shape, 10, 1, 0.9, 1.0)
        n, P = 32 ** 3, f0.descriptor.padded_sites
        for got, ref in ((f1.data, of), (g1.data, og)):
            rel = np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300))
            assert rel <= 1e-12, rel
        rho_g = f1.data.reshape(19, P)[:, :n].sum(0)
        rho_r = of.reshape(19, P)[:, :n].sum(0)
        phi_g = g1.data.reshape(19, P)[:, :n].sum(0)
        phi_r = og.reshape(19, P)[:, :n].sum(0)
        assert np.max(np.abs(rho_g - rho_r) / np.abs(rho_r)) <= 1e-12
        assert np.max(np.abs(phi_g - phi_r) / np.maximum(np.abs(phi_r), 1e-3)) <= 1e-12

    def test_passive_equals_reference_collision_after_streaming(self, lk, golden):
        from oracle import oracle as orc

        shape = (8, 8, 8)
        f0, g0 = _state(lk, shape, 5)
        with lk.BinaryFluid(lk.LatticeShape(*shape), physics="passive") as sim:
            sim.load(f0, g0)
            sim.run(1)
            f1, g1 = sim.fields()
        P = f0.descriptor.padded_sites
        fs, gs = orc.stream_numpy(f0.data, shape, P), orc.stream_numpy(g0.data, shape, P)
        orc.collide(fs, gs, P, 512)
        assert np.array_equal(f1.data, fs) and np.array_equal(g1.data, gs)

    def test_singular_state_raises(self, lk):
        shape = (8, 8, 4)
        f0, g0 = _state(lk, shape, 1)
        f0.data[:] = 0.0
        with lk.BinaryFluid(lk.LatticeShape(*shape)) as sim:
            sim.load(f0, g0)
            sim.run(1)
            with pytest.raises(lk.SingularStateError):
                sim.sync()

    @pytest.mark.parametrize("physics", ["binary", "passive", "binary-stress"])
    @pytest.mark.parametrize("layout", ["row", "soa"])
    def test_nccl_self_exchange_matches_oracle(self, lk, physics, layout):
        # the NCCL slab path at P = 1 (a self communicator): packed f/g faces,
        # phi and two-plane mu faces, in both f/g layouts
        if not lk.nccl_available():
            pytest.skip("libnccl.so.2 not loadable")
        shape = (16, 8, 8)
        f0, g0 = _state(lk, shape, 13)
        with lk.BinaryFluid(lk.LatticeShape(*shape), physics=physics, use_graph=False) as sim:
            sim.set_layout(lk.LAYOUT_ROW if layout == "row" else lk.LAYOUT_SOA)
            sim.attach_nccl(lk.nccl_unique_id())
            sim.load(f0, g0)
            sim.run(3)
            f1, g1 = sim.fields()
        code = {"passive": 0, "binary": 1, "binary-stress": 2}[physics]
        of, og, _, _ = _oracle(f0, g0, shape, 3, code)
        assert np.array_equal(f1.data, of) and np.array_equal(g1.data, og)

    def test_reload_between_runs(self, lk):
        shape = (16, 16, 8)
        f0, g0 = _state(lk, shape, 3)
        f1, g1 = _state(lk, shape, 4)
        with lk.BinaryFluid(lk.LatticeShape(*shape)) as sim:
            sim.load(f0, g0)
            sim.run(2)
            sim.load(f1, g1)
            sim.run(3)
            fa, ga = sim.fields()
        of, og, _, _ = _oracle(f1, g1, shape, 3, 1)
        assert np.array_equal(fa.data, of) and np.array_equal(ga.data, og)

    def test_errors_stay_with_their_engine(self, lk):
        # two engines on one GPU: only the singular one raises at its sync
        shape = (8, 8, 4)
        fa, ga = _state(lk, shape, 1)
        fb, gb = _state(lk, shape, 2)
        fa.data[:] = 0.0
        with lk.BinaryFluid(lk.LatticeShape(*shape)) as a, \
                lk.BinaryFluid(lk.LatticeShape(*shape)) as b:
            a.load(fa, ga)
            b.load(fb, gb)
            a.run(1)
            b.run(1)
            b.sync()                      # clean
            with pytest.raises(lk.SingularStateError):
                a.sync()
            a.sync()                      # reported once, then cleared
            b.sync()


class TestStressForm:
    """physics "binary-stress": the force as the divergence of the chemical
    pressure tensor (mu kernels also write p_iso and grad phi; collide-stream
    differentiates them).  Bitwise vs the oracle in EXACT mode."""

    @pytest.mark.parametrize("shape", [(16, 12, 10), (32, 16, 6), (7, 6, 5), (64, 8, 9)])
    @pytest.mark.parametrize("graph", [True, False])
    def test_exact_bitwise(self, lk, shape, graph):
        f0, g0 = _state(lk, shape, 23)
        model = lk.D3Q19Model(tau_f=0.8, tau_g=1.1)
        with lk.BinaryFluid(lk.LatticeShape(*shape), model=model, physics="binary-stress",
                            use_graph=graph) as sim:
            sim.load(f0, g0)
            sim.run(4)
            f1, g1 = sim.fields()
        of, og, _, _ = _oracle(f0, g0, shape, 4, 2, 0.8, 1.1)
        assert np.array_equal(f1.data.view(np.uint64), of.view(np.uint64))
        assert np.array_equal(g1.data.view(np.uint64), og.view(np.uint64))

    def test_vvl2_exact_bitwise(self, lk):
        shape = (16, 8, 8)
        f0, g0 = _state(lk, shape, 5)
        with lk.BinaryFluid(lk.LatticeShape(*shape), physics="binary-stress", vvl=2) as sim:
            sim.load(f0, g0)
            sim.run(3)
            f1, g1 = sim.fields()
        of, og, _, _ = _oracle(f0, g0, shape, 3, 2)
        assert np.array_equal(f1.data, of) and np.array_equal(g1.data, og)

    def test_fast_within_1e12_and_momentum(self, lk):
        shape = (32, 32, 32)
        f0, g0 = _state(lk, shape, 11)
        with lk.BinaryFluid(lk.LatticeShape(*shape), mode=lk.MODE_FAST,
                            physics="binary-stress") as sim:
            sim.load(f0, g0)
            t0 = sim.totals()
            sim.run(10)
            t1 = sim.totals()
            f1, g1 = sim.fields()
        of, og, _, _ = _oracle(f0, g0, shape, 10, 2)
        for got, ref in ((f1.data, of), (g1.data, og)):
            rel = np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300))
            assert rel <= 1e-12, rel
        assert np.allclose(t1[1:4], t0[1:4], rtol=0, atol=1e-11)   # momentum conserved

    def test_nccl_self_exchange(self, lk):
        if not lk.nccl_available():
            pytest.skip("libnccl.so.2 not loadable")
        shape = (16, 8, 8)
        f0, g0 = _state(lk, shape, 13)
        with lk.BinaryFluid(lk.LatticeShape(*shape), physics="binary-stress",
                            use_graph=False) as sim:
            sim.attach_nccl(lk.nccl_unique_id())
            sim.load(f0, g0)
            sim.run(3)
            f1, g1 = sim.fields()
        of, og, _, _ = _oracle(f0, g0, shape, 3, 2)
        assert np.array_equal(f1.data, of) and np.array_equal(g1.data, og)


class TestSpinodalPhysics:
    """A symmetric mixture (phi = 0 +- 0.01) phase-separates: |phi| grows toward
    phi* = 1, the discrete free energy decreases at every checkpoint, total phi
    and mass stay conserved -- for both force forms (long-run behaviour:
    profiles/r01_spinodal_*.txt)."""

    @pytest.mark.parametrize("physics", ["binary", "binary-stress"])
    def test_phase_separation(self, lk, physics):
        from paper_1405_6162_b200.lattice import FieldDescriptor, field_create

        N = 32
        fe, model = lk.FreeEnergy(), lk.D3Q19Model()
        shape = lk.LatticeShape(N, N, N)
        desc = FieldDescriptor.create(19, shape.nsites)
        f, g = field_create(desc), field_create(desc)
        phi0 = 0.01 * (2 * np.random.default_rng(3).random(shape.nsites) - 1)
        for i in range(19):
            f.component(i)[:] = model.wv[i]
            g.component(i)[:] = model.wv[i] * phi0
        n, P = shape.nsites, desc.padded_sites

        def energy(gd):
            phi = gd.reshape(19, P)[:, :n].sum(0).reshape(N, N, N)
            grad = [(np.roll(phi, -1, a) - np.roll(phi, 1, a)) * 0.5 for a in range(3)]
            return (float(np.sum(0.5 * fe.A * phi ** 2 + 0.25 * fe.B * phi ** 4
                                 + 0.5 * fe.kappa * sum(x * x for x in grad))),
                    float(np.abs(phi).mean()))

        with lk.BinaryFluid(shape, model=model, free_energy=fe, physics=physics,
                            mode=lk.MODE_FAST) as sim:
            sim.load(f, g)
            t0 = sim.totals()
            hist = []
            for _ in range(12):
                sim.run(100)
                hist.append(energy(sim.fields()[1].data))
            t1 = sim.totals()
        energies = [h[0] for h in hist]
        assert all(b < a for a, b in zip(energies, energies[1:])), energies
        assert hist[-1][1] > 0.6                      # domains forming toward phi* = +-1
        assert abs(t1[0] - t0[0]) <= 1e-12 * t0[0]
        assert abs(t1[4] - t0[4]) <= 1e-10


class TestSlabDecomposition:
    """P virtual slabs on one GPU, halos moved with the C-ABI face/plane calls."""

    @pytest.mark.parametrize("nslabs", [2, 4])
    def test_slabs_bitwise_equal_single(self, lk, nslabs):
        from paper_1405_6162_b200 import _native as nat
        from paper_1405_6162_b200.fluid import fluid_params
        from paper_1405_6162_b200.slabs import VirtualSlabs

        shape = (12, 8, 16)
        f0, g0 = _state(lk, shape, 21)
        vs = VirtualSlabs(lk.LatticeShape(*shape), nslabs, fluid_params())
        vs.load(f0, g0)
        vs.run(3)
        f1, g1 = vs.fields()
        vs.close()
        of, og, _, _ = _oracle(f0, g0, shape, 3, 1)
        assert np.array_equal(f1.data, of) and np.array_equal(g1.data, og)


class TestFullSizeProperties:
    """BASELINE sizes through size-independent properties (north-star tolerance)."""

    def test_256cube_exact_vs_oracle_and_fast(self, lk):
        # configs[2]: one EXACT step bitwise vs the oracle, FAST within 1e-12
        shape = (256, 256, 256)
        f0, g0 = _state(lk, shape, 1234)
        ex = {}
        for mode in (lk.MODE_EXACT, lk.MODE_FAST):
            with lk.BinaryFluid(lk.LatticeShape(*shape), mode=mode) as sim:
                sim.load(f0, g0)
                sim.run(2)
                ex[mode] = sim.fields()
        of, og, _, _ = _oracle(f0, g0, shape, 2, 1)
        assert np.array_equal(ex[lk.MODE_EXACT][0].data, of)
        assert np.array_equal(ex[lk.MODE_EXACT][1].data, og)
        for got, ref in ((ex[lk.MODE_FAST][0].data, of), (ex[lk.MODE_FAST][1].data, og)):
            rel = np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300))
            assert rel <= 1e-12, rel

    def test_256_plane_stress_form_exact_vs_oracle(self, lk):
        # the stress form at the BASELINE plane size: two EXACT steps bitwise
        shape = (256, 256, 32)
        f0, g0 = _state(lk, shape, 77)
        with lk.BinaryFluid(lk.LatticeShape(*shape), physics="binary-stress") as sim:
            sim.load(f0, g0)
            sim.run(2)
            f1, g1 = sim.fields()
        of, og, _, _ = _oracle(f0, g0, shape, 2, 2)
        assert np.array_equal(f1.data, of) and np.array_equal(g1.data, og)

    def test_256cube_long_run_conservation(self, lk):
        # 200 FAST steps: total mass and total phi conserved to rounding
        shape = lk.LatticeShape(256, 256, 256)
        f0, g0 = _state(lk, (256, 256, 256), 99)
        n, P = shape.nsites, f0.descriptor.padded_sites
        m0 = f0.data.reshape(19, P)[:, :n].sum(dtype=np.float64)
        p0 = g0.data.reshape(19, P)[:, :n].sum(dtype=np.float64)
        with lk.BinaryFluid(shape, mode=lk.MODE_FAST) as sim:
            sim.load(f0, g0)
            sim.run(200)
            f1, g1 = sim.fields()
        m1 = f1.data.reshape(19, P)[:, :n].sum(dtype=np.float64)
        p1 = g1.data.reshape(19, P)[:, :n].sum(dtype=np.float64)
        assert abs(m1 - m0) <= 1e-10 * abs(m0)
        assert abs(p1 - p0) <= 1e-10 * abs(p0)
        assert np.all(np.isfinite(f1.data)) and np.all(np.isfinite(g1.data))

    def test_totals_match_fields(self, lk):
        shape = lk.LatticeShape(64, 32, 48)
        f0, g0 = _state(lk, (64, 32, 48), 4)
        with lk.BinaryFluid(shape, mode=lk.MODE_FAST) as sim:
            sim.load(f0, g0)
            t0 = sim.totals()
            sim.run(10)
            t1 = sim.totals()
            f1, g1 = sim.fields()
        n, P = shape.nsites, f0.descriptor.padded_sites
        fc = f1.data.reshape(19, P)[:, :n]
        cv = lk.D3Q19Model().cvf
        ref = [fc.sum(), (cv[:, 0] @ fc).sum(), (cv[:, 1] @ fc).sum(), (cv[:, 2] @ fc).sum(),
               g1.data.reshape(19, P)[:, :n].sum()]
        assert np.allclose(t1, ref, rtol=1e-12, atol=1e-9)
        assert abs(t1[0] - t0[0]) <= 1e-12 * t0[0]      # mass conserved
        assert abs(t1[4] - t0[4]) <= 1e-12 * abs(t0[4])  # phi conserved

    def test_ragged_shapes(self, lk):
        # odd extents, nx not a multiple of the warp, planes of odd size, nz = 1
        for shape in ((7, 6, 5), (33, 10, 3), (2, 2, 2), (64, 3, 9), (8, 4, 1), (1, 2, 3)):
            f0, g0 = _state(lk, shape, 5)
            with lk.BinaryFluid(lk.LatticeShape(*shape)) as sim:
                sim.load(f0, g0)
                sim.run(3)
                f1, g1 = sim.fields()
            of, og, _, _ = _oracle(f0, g0, shape, 3, 1)
            assert np.array_equal(f1.data, of) and np.array_equal(g1.data, og), shape

    def test_odd_plane_rejected(self, lk):
        with pytest.raises(lk.ShapeError):
            lk.BinaryFluid(lk.LatticeShape(3, 5, 4))


class TestStencilKernels:
    """The C-ABI stencil launchers against the oracle on random phi slabs, for
    both mu kernels: the shared-memory tile kernel k_mu_tile (nx % 32 == 0,
    ny % 8 == 0; elsewhere the plain kernel runs) and the plain k_mu."""

    @pytest.mark.parametrize("shape", [(256, 16, 37), (32, 8, 16), (2, 8, 5), (512, 24, 3),
                                       (30, 16, 18), (12, 12, 7), (64, 8, 1), (96, 40, 17)])
    @pytest.mark.parametrize("variant", [0, 1])
    def test_mu_matches_oracle(self, lk, shape, variant):
        prev = lk.mu_variant(variant)
        try:
            self._check_mu(lk, shape)
        finally:
            lk.mu_variant(prev)

    def _check_mu(self, lk, shape):
        import ctypes

        from oracle import oracle as orc
        from paper_1405_6162_b200 import _native as nat
        from paper_1405_6162_b200.fluid import fluid_params

        nx, ny, nz = shape
        PL = nx * ny
        rng = np.random.default_rng(nz)
        phi_host = rng.random((nz, ny, nx)) * 2 - 1            # device order (z, y, x)
        buf = np.zeros((nz + 2, ny, nx))
        buf[1:nz + 1] = phi_host
        buf[0], buf[nz + 1] = phi_host[nz - 1], phi_host[0]   # periodic halos
        slab = nat.Slab(nx, ny, nz, -(-((nz + 2) * PL) // 64) * 64)
        mu_planes = np.zeros((nz + 4, ny, nx))                 # mu layout: zs = z + 2
        d_phi, d_mu = nat.malloc(buf.nbytes), nat.malloc(mu_planes.nbytes)
        try:
            nat.check(nat.lib.ltk_h2d(d_phi, buf.ctypes.data, buf.nbytes, None))
            prm = fluid_params()
            for lo, hi in ((0, nz), (1, max(1, nz - 1))):
                nat.check(nat.lib.ltk_fluid_mu(ctypes.byref(slab), d_phi, d_mu, ctypes.byref(prm),
                                               lo, hi, None))
                out = np.zeros_like(mu_planes)
                nat.check(nat.lib.ltk_d2h(out.ctypes.data, d_mu, out.nbytes, None))
                nat.check(nat.lib.ltk_stream_sync(None))
                ref = np.zeros(nx * ny * nz)
                ph = np.ascontiguousarray(phi_host.transpose(2, 1, 0)).ravel()   # host (x, y, z)
                orc.lib().orc_mu(orc._p(ph), orc._p(ref), nx, ny, nz, prm.A, prm.B, prm.kappa)
                ref_dev = ref.reshape(nx, ny, nz).transpose(2, 1, 0)
                assert np.array_equal(out[2 + lo:2 + hi], ref_dev[lo:hi]), (shape, lo, hi)
        finally:
            nat.free(d_phi)
            nat.free(d_mu)


class TestRandomShapes:
    """Hypothesis-driven parity: random lattice shapes (nx*ny even, the engine's
    16-byte row rule; some multiples of 32 x 8 so the register mu kernel runs),
    physics, tau, step counts and f/g layout, EXACT bitwise vs the oracle.
    LTK_HYP_EXAMPLES raises the example count (default 30)."""

    def test_random_shapes_bitwise(self, lk):
        from hypothesis import given, settings
        from hypothesis import strategies as st

        @settings(max_examples=int(os.environ.get("LTK_HYP_EXAMPLES", "30")), deadline=None)
        @given(nx=st.one_of(st.integers(1, 12), st.sampled_from([32, 64])),
               ny=st.one_of(st.integers(1, 12), st.sampled_from([8, 16])),
               nz=st.integers(1, 9),
               physics=st.sampled_from(["passive", "binary", "binary-stress"]),
               tau=st.sampled_from([(1.0, 1.0), (0.8, 1.3), (1.6, 0.7)]),
               steps=st.integers(1, 3), seed=st.integers(0, 10 ** 6),
               row=st.booleans())
        def check(nx, ny, nz, physics, tau, steps, seed, row):
            seen.append((nx, ny, nz, physics, row))
            if (nx * ny) % 2:
                nx += 1
            shape = (nx, ny, nz)
            f0, g0 = _state(lk, shape, seed)
            model = lk.D3Q19Model(tau_f=tau[0], tau_g=tau[1])
            with lk.BinaryFluid(lk.LatticeShape(*shape), model=model, physics=physics) as sim:
                sim.set_layout(lk.LAYOUT_ROW if row and nx % 2 == 0 else lk.LAYOUT_SOA)
                sim.load(f0, g0)
                sim.run(steps)
                f1, g1 = sim.fields()
            code = {"passive": 0, "binary": 1, "binary-stress": 2}[physics]
            of, og, _, _ = _oracle(f0, g0, shape, steps, code, tau[0], tau[1])
            assert np.array_equal(f1.data.view(np.uint64), of.view(np.uint64)), shape
            assert np.array_equal(g1.data.view(np.uint64), og.view(np.uint64)), shape

        seen = []
        check()
        print(f"random-shape parity: {len(seen)} examples, "
              f"{sum(1 for c in seen if c[0] % 32 == 0 and c[1] % 8 == 0)} on the k_mu_tile path, "
              f"{sum(1 for c in seen if c[4])} row-blocked")


class TestRowLayout:
    """The engine's row-blocked f/g layout (LTK_LAYOUT_ROW: the 19 components
    of an x-row adjacent) against the SoA layout and the oracle: bitwise for
    every physics, mode, VVL and graph on/off; load/store, totals and the
    periodic images go through the same strides."""

    @staticmethod
    def _run(lk, shape, layout, physics="binary", mode=None, vvl=1, graph=True, steps=4,
             seed=23):
        f0, g0 = _state(lk, shape, seed)
        model = lk.D3Q19Model(tau_f=0.9, tau_g=1.2)
        mode = lk.MODE_EXACT if mode is None else mode
        with lk.BinaryFluid(lk.LatticeShape(*shape), model=model, physics=physics, mode=mode,
                            vvl=vvl, use_graph=graph) as sim:
            default = lk.LAYOUT_SOA if os.environ.get("LTK_LAYOUT") == "0" else lk.LAYOUT_ROW
            assert sim.set_layout(layout) == default  # row-blocked for even nx
            assert sim.set_layout(None) == layout
            sim.load(f0, g0)
            sim.run(steps)
            f1, g1 = sim.fields()
            phi, mu = sim.order_parameter()
            tot = sim.totals()
        return f0, g0, (f1.data, g1.data, phi, mu, tot)

    @pytest.mark.parametrize("physics", ["binary", "passive", "binary-stress"])
    @pytest.mark.parametrize("shape", [(16, 12, 10), (32, 16, 6), (6, 10, 4), (64, 3, 9)])
    def test_row_matches_oracle(self, lk, shape, physics):
        f0, g0, got = self._run(lk, shape, lk.LAYOUT_ROW, physics)
        ph = {"passive": 0, "binary": 1, "binary-stress": 2}[physics]
        of, og, _, _ = _oracle(f0, g0, shape, 4, ph, 0.9, 1.2)
        assert np.array_equal(got[0].view(np.uint64), of.view(np.uint64))
        assert np.array_equal(got[1].view(np.uint64), og.view(np.uint64))

    @pytest.mark.parametrize("physics", ["binary", "binary-stress"])
    @pytest.mark.parametrize("vvl,graph", [(1, False), (2, True)])
    def test_row_equals_soa(self, lk, physics, vvl, graph):
        shape = (32, 12, 14)
        for mode in (lk.MODE_EXACT, lk.MODE_FAST):
            _, _, ref = self._run(lk, shape, lk.LAYOUT_SOA, physics, mode, vvl, graph)
            _, _, got = self._run(lk, shape, lk.LAYOUT_ROW, physics, mode, vvl, graph)
            for a, b in zip(got, ref):
                assert np.array_equal(np.asarray(a).view(np.uint64),
                                      np.asarray(b).view(np.uint64)), (mode, vvl, graph)

    def test_row_large_plane_fast(self, lk):
        # BASELINE plane size
        shape = (256, 256, 12)
        _, _, got = self._run(lk, shape, lk.LAYOUT_ROW, mode=lk.MODE_FAST, steps=3)
        _, _, ref = self._run(lk, shape, lk.LAYOUT_SOA, mode=lk.MODE_FAST, steps=3)
        for a, b in zip(got, ref):
            assert np.array_equal(a, b)

    def test_row_layout_rules(self, lk):
        with lk.BinaryFluid(lk.LatticeShape(7, 4, 4)) as sim:
            assert sim.set_layout(None) == lk.LAYOUT_SOA  # odd nx keeps SoA
            with pytest.raises(lk.ShapeError):
                sim.set_layout(lk.LAYOUT_ROW)  # odd nx
            with pytest.raises(lk.ConfigError):
                sim.set_layout(5)
        a = lk.BinaryFluid(lk.LatticeShape(16, 4, 8), rank=0, nranks=2)
        b = lk.BinaryFluid(lk.LatticeShape(16, 4, 8), rank=1, nranks=2)
        try:
            a.set_layout(lk.LAYOUT_SOA)
            b.set_layout(lk.LAYOUT_ROW)
            with pytest.raises(lk.ShapeError):
                a.attach_peer_engines(b, b)  # layouts differ
            a.set_layout(lk.LAYOUT_ROW)
            a.attach_peer_engines(b, b)
            with pytest.raises(lk.ConfigError):
                a.set_layout(lk.LAYOUT_SOA)  # after attaching a transport
        finally:
            a.close()
            b.close()
