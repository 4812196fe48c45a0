"""Host-side API mirror (CPU): lattice, model, constants, plans, schedules.

Mirrors reference tests test_lattice.py, test_model.py and the plan parts of
test_execution.py / test_memory.py that do not need a device.
"""

import io

import numpy as np
import pytest

import paper_1405_6162_b200 as lk
from paper_1405_6162_b200.memory import ConstantBlock
from paper_1405_6162_b200.model import CZ_DOWN, CZ_UP, Q


class TestLattice:
    def test_soa_index(self):
        assert lk.soa_index(0, 0, 100) == 0
        assert lk.soa_index(1, 5, 100) == 105
        assert lk.soa_index(18, 7, 8, ncomp=19) == 151
        with pytest.raises(lk.BoundsError):
            lk.soa_index(0, 8, 8)
        with pytest.raises(lk.BoundsError):
            lk.soa_index(3, 0, 8, ncomp=3)

    def test_pad_sites(self):
        assert lk.pad_sites(64, 8) == 64 and lk.pad_sites(65, 8) == 72 and lk.pad_sites(1, 4) == 4
        with pytest.raises(lk.ConfigError):
            lk.pad_sites(64, 0)
        for n in range(1, 200):
            for v in (1, 2, 3, 8, 16):
                p = lk.pad_sites(n, v)
                assert p >= n and p % v == 0 and p - n < v

    def test_shape(self):
        assert lk.LatticeShape(4, 5, 6).nsites == 120
        assert lk.LatticeShape.parse("16x8x4") == lk.LatticeShape(16, 8, 4)
        for bad in ("16x8", "axbxc"):
            with pytest.raises(lk.ConfigError):
                lk.LatticeShape.parse(bad)
        with pytest.raises(lk.ConfigError):
            lk.LatticeShape(0, 1, 1)

    def test_field_and_diff(self):
        desc = lk.FieldDescriptor.create(1, 5, max_vvl=8)
        a, b = lk.field_create(desc), lk.field_create(desc)
        b.data[5:] = 99.0
        assert lk.field_max_abs_diff(a, b) == 0.0
        with pytest.raises(lk.ShapeError):
            lk.field_max_abs_diff(a, lk.field_create(lk.FieldDescriptor.create(2, 5)))

    def test_aos_soa(self):
        desc = lk.FieldDescriptor.create(2, 2, max_vvl=2)
        f = lk.aos_to_soa(np.array([1.0, 10.0, 2.0, 20.0]), desc)
        assert list(f.data) == [1.0, 2.0, 10.0, 20.0]
        flat = np.random.default_rng(0).random(3 * 7)
        assert np.array_equal(lk.soa_to_aos(lk.aos_to_soa(flat, lk.FieldDescriptor.create(3, 7))),
                              flat)

    def test_dump_load(self):
        shape = lk.LatticeShape(3, 4, 5)
        desc = lk.FieldDescriptor.create(3, shape.nsites)
        f = lk.field_create(desc)
        f.data[:] = np.random.default_rng(7).random(desc.nelem)
        f.components()[:, shape.nsites:] = 0
        buf = io.BytesIO()
        lk.field_dump(f, shape, buf)
        assert len(buf.getvalue()) == 32 + 8 * 3 * shape.nsites
        buf.seek(0)
        g, shape2 = lk.field_load(buf)
        assert shape2 == shape and lk.field_max_abs_diff(f, g) == 0.0
        with pytest.raises(lk.ShapeError):
            lk.field_load(io.BytesIO(b"\x00" * 10))


class TestModel:
    def test_velocity_set_and_weights(self):
        m = lk.D3Q19Model()
        nz = np.count_nonzero(m.cv, axis=1)
        assert list(nz).count(0) == 1 and list(nz).count(1) == 6 and list(nz).count(2) == 12
        assert np.array_equal(m.cv[m.negation_index()], -m.cv)
        assert m.wv[0] == 1.0 / 3.0

    def test_moment_identities(self):
        m = lk.D3Q19Model()
        assert abs(sum(m.wv) - 1.0) <= 1e-15
        for a in range(3):
            assert abs(sum(m.wv[i] * m.cv[i, a] for i in range(Q))) <= 1e-15
            for b in range(3):
                s = sum(m.wv[i] * m.cv[i, a] * m.cv[i, b] for i in range(Q))
                assert abs(s - (m.cs2 if a == b else 0.0)) <= 1e-15

    def test_tau_validation(self):
        with pytest.raises(lk.ConfigError):
            lk.D3Q19Model(tau_f=0.5)

    def test_crossing_sets(self):
        assert CZ_UP == (5, 11, 13, 15, 17) and CZ_DOWN == (6, 12, 14, 16, 18)

    def test_site_ops_match_reference_vectors(self, golden):
        _, small = golden
        m = lk.D3Q19Model()
        rho, u = lk.moments(m.wv, m)
        assert np.array_equal(np.array([rho, *u]), small["site_moments_wv"])
        assert np.array_equal(lk.equilibrium(1.2, (0.03, -0.05, 0.02), m), small["site_equilibrium"])
        f = small["site_relax_in"]
        r, uu = lk.moments(f, m)
        assert np.array_equal(lk.bgk_relax(f, lk.equilibrium(r, uu, m), 0.8),
                              small["site_relax_out"])


class TestConstantsAndPlans:
    def test_constant_store(self):
        cb = ConstantBlock()
        src = np.array([1.0, 2.0, 3.0])
        cb.set_double_array("v", src, (3,))
        src[:] = -1
        assert list(cb.get("v")) == [1.0, 2.0, 3.0]
        cb.set_double("x", 1.0)
        with pytest.raises(lk.TypeConflictError):
            cb.set_int("x", 1)
        cb.set_int_array("iv", [1, 2, 3], (3,))
        cb.set_double_array("m", np.arange(6.0), (2, 3))
        assert cb.get("m").shape == (2, 3)

    def test_launch_plan(self):
        assert lk.LaunchPlan(extent=64, vvl=8).chunk_count == 8
        with pytest.raises(lk.PlanError):
            lk.LaunchPlan(extent=64, vvl=5)
        with pytest.raises(lk.PlanError):
            lk.LaunchPlan(extent=8, vvl=0)
        p = lk.LaunchPlan(extent=2 ** 21, vvl=2, tpb=128)
        assert p.cuda_grid == 2 ** 20 // 128 and p.cuda_block == 128
        assert lk.LaunchPlan(extent=64, vvl=8, tpb=4).cuda_block == 32

    def test_schedule_partitions_chunks(self):
        for tpb in (1, 32, 100, 256):
            plan = lk.LaunchPlan(extent=112 * 16, vvl=8, tpb=tpb)
            covered = [c for blk in lk.backend_schedule(plan) for lo, hi in blk
                       for c in range(lo, hi)]
            assert covered == list(range(plan.chunk_count))

    def test_reference_backend_schedules(self):
        # the reference's own expectations (reference tests/test_execution.py:44-72)
        P = lk.LaunchPlan
        assert lk.backend_schedule(P(extent=64, vvl=8, workers=2), "threaded") == \
            [[(0, 4)], [(4, 8)]]
        assert lk.backend_schedule(P(extent=64, vvl=8, workers=1), "threaded") == [[(0, 8)]]
        assert lk.backend_schedule(P(extent=56, vvl=8, workers=2), "threaded") == \
            [[(0, 4)], [(4, 7)]]
        assert lk.backend_schedule(P(extent=64, vvl=8), "reference") == [[(0, 8)]]
        sched = lk.backend_schedule(P(extent=64, vvl=8, workers=2, tpb=4), "emulated")
        assert sorted(r for w in sched for r in w) == [(0, 4), (4, 8)]
        for backend in ("reference", "threaded", "emulated", "cuda"):
            for workers in (1, 2, 3, 5):
                plan = P(extent=112, vvl=8, workers=workers, tpb=3)
                covered = sorted(c for w in lk.backend_schedule(plan, backend)
                                 for lo, hi in w for c in range(lo, hi))
                assert covered == list(range(plan.chunk_count))
        with pytest.raises(lk.PlanError):
            lk.backend_schedule(P(extent=64, vvl=8), "bogus")


class TestSlabSchedule:
    @pytest.mark.parametrize("nranks", [1, 2, 3, 8])
    def test_schedule_matches_pairwise(self, nranks):
        from paper_1405_6162_b200.slabs import match_schedules

        for kind in ("fg", "phi", "mu"):
            pairs = match_schedules(nranks, 4, kind)
            assert len(pairs) == nranks * (20 if kind == "fg" else 2)
            for send, receiver, recv in pairs:
                # the top owned plane(s) land in the receiver's bottom halo(s) and vice
                # versa; mu moves two planes per face (mu layout zs = z + 2)
                ok = ((4, 0), (2, 6)) if kind == "mu" else ((4, 0), (1, 5))
                assert (send.plane, recv.plane) in ok

    def test_slab_bounds(self):
        from paper_1405_6162_b200.slabs import slab_bounds

        assert slab_bounds(512, 3, 8) == (192, 64)
        with pytest.raises(lk.ShapeError):
            slab_bounds(10, 0, 3)
