"""GPU parity of the reference hot path: the D3Q19 binary collision through
the reference-facing API (TargetDevice / launch / sync_target -> ltk_collide).

Bar: bitwise equal to the reference (EXACT mode) on the golden vectors that
the reference itself produced (tests/golden/), and to the oracle on fresh
inputs; FAST mode within 1e-12 relative.  Reference tests mirrored:
test_kernels.py:157-214, test_acceptance.py:56-101.
"""

import hashlib

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


@pytest.fixture(scope="module")
def lk():
    import paper_1405_6162_b200 as lk

    return lk


def _state(lk, shape, seed, model=None):
    from paper_1405_6162_b200.kernels import random_binary_state

    return random_binary_state(lk.LatticeShape(*shape), np.random.default_rng(seed),
                               model or lk.D3Q19Model())


class TestGoldenParity:
    @pytest.mark.parametrize("vvl", [1, 2, 4, 8, 16])
    def test_all_golden_cases_bitwise(self, lk, golden, vvl):
        from paper_1405_6162_b200.verify import run_framework_collision

        meta, _ = golden
        for case in meta["collision"]:
            if case["padded"] % vvl:
                continue
            model = lk.D3Q19Model(tau_f=case["tau_f"], tau_g=case["tau_g"])
            f0, g0 = _state(lk, case["shape"], case["seed"], model)
            assert sha(f0.data) == case["in_f"]
            f1, g1 = run_framework_collision(f0, g0, "cuda", vvl, 1, steps=case["steps"],
                                             model=model)
            if sha(f1.data) != case["out_f"] or sha(g1.data) != case["out_g"]:
                from oracle import oracle as orc

                rf, rg = f0.data.copy(), g0.data.copy()
                P = f0.descriptor.padded_sites
                orc.collide(rf, rg, P, f0.descriptor.nsites, tau_f=case["tau_f"],
                            tau_g=case["tau_g"], steps=case["steps"])
                bad = np.flatnonzero(f1.data.view(np.uint64) != rf.view(np.uint64))
                ulp = f1.data.view(np.int64)[bad] - rf.view(np.int64)[bad]
                raise AssertionError(f"{case['shape']} vvl={vvl}: {bad.size} f elements differ, "
                                     f"sites {np.unique(bad % P)[:10]}, comps "
                                     f"{np.unique(bad // P)}, ulps {np.unique(ulp)[:10]}")

    @pytest.mark.parametrize("tpb", [32, 64, 256])
    def test_tpb_independent(self, lk, golden, tpb):
        from paper_1405_6162_b200.verify import run_framework_collision

        meta, _ = golden
        case = meta["collision"][2]  # 16^3
        model = lk.D3Q19Model(tau_f=case["tau_f"], tau_g=case["tau_g"])
        f0, g0 = _state(lk, case["shape"], case["seed"], model)
        f1, g1 = run_framework_collision(f0, g0, "cuda", 2, 1, steps=case["steps"], model=model,
                                         tpb=tpb)
        assert sha(f1.data) == case["out_f"] and sha(g1.data) == case["out_g"]

    def test_fast_mode_within_1e12(self, lk):
        from oracle import oracle as orc
        from paper_1405_6162_b200.verify import run_framework_collision

        model = lk.D3Q19Model(tau_f=0.8, tau_g=1.3)
        f0, g0 = _state(lk, (32, 32, 32), 99, model)
        f1, g1 = run_framework_collision(f0, g0, "cuda", 2, 1, steps=10, model=model,
                                         mode=lk.MODE_FAST)
        rf, rg = f0.data.copy(), g0.data.copy()
        orc.collide(rf, rg, f0.descriptor.padded_sites, 32 ** 3, tau_f=0.8, tau_g=1.3, steps=10)
        for got, ref in ((f1.data, rf), (g1.data, rg)):
            rel = np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300))
            assert rel <= 1e-12, rel

    def test_large_lattice_bitwise_vs_oracle(self, lk):
        # 128^3, BASELINE configs[1], against the oracle (itself pinned bitwise)
        from oracle import oracle as orc
        from paper_1405_6162_b200.verify import run_framework_collision

        model = lk.D3Q19Model(tau_f=0.8, tau_g=1.0)
        f0, g0 = _state(lk, (128, 128, 128), 1234, model)
        f1, g1 = run_framework_collision(f0, g0, "cuda", 1, 1, steps=2, model=model)
        rf, rg = f0.data.copy(), g0.data.copy()
        orc.collide(rf, rg, f0.descriptor.padded_sites, 128 ** 3, tau_f=0.8, tau_g=1.0, steps=2,
                    threads=8)
        assert np.array_equal(f1.data, rf) and np.array_equal(g1.data, rg)


class TestContracts:
    def test_singular_state_surfaces_at_sync(self, lk):
        # reference test_kernels.py:187-197
        desc = lk.FieldDescriptor.create(19, 8, max_vvl=8)
        dev = lk.TargetDevice()
        lk.set_model_constants(dev, lk.D3Q19Model())
        bf, bg = lk.target_malloc(dev, desc), lk.target_malloc(dev, desc)
        lk.launch(dev, lk.binary_collision_kernel, lk.LaunchPlan(extent=desc.padded_sites, vvl=8),
                  [bf, bg])
        with pytest.raises(lk.SingularStateError):
            lk.sync_target(dev)
        lk.sync_target(dev)  # error consumed

    def test_padding_untouched(self, lk):
        from paper_1405_6162_b200.verify import run_framework_collision

        f0, g0 = _state(lk, (3, 3, 3), 6)
        for vvl in (1, 2, 4, 8, 16):
            f1, g1 = run_framework_collision(f0, g0, "cuda", vvl, 1)
            P = f0.descriptor.padded_sites
            for i in range(19):
                assert not f1.data[i * P + 27:(i + 1) * P].any()
                assert not g1.data[i * P + 27:(i + 1) * P].any()

    def test_equilibrium_fixed_point_and_conservation(self, lk):
        from paper_1405_6162_b200.verify import verify_conservation, verify_fixed_point

        ok, lines = verify_fixed_point(lk.LatticeShape(8, 8, 8))
        assert ok, lines
        ok, lines = verify_conservation(lk.LatticeShape(16, 16, 16), seed=20140709)
        assert ok, lines

    def test_verify_suite(self, lk):
        from paper_1405_6162_b200.verify import run_verify_suite

        ok, lines = run_verify_suite("binary-collision", lk.LatticeShape(8, 8, 8))
        assert ok, lines

    def test_descriptor_mismatch_and_missing_constant(self, lk):
        dev = lk.TargetDevice()
        lk.set_model_constants(dev, lk.D3Q19Model())
        bf = lk.target_malloc(dev, lk.FieldDescriptor.create(19, 16))
        bg = lk.target_malloc(dev, lk.FieldDescriptor.create(19, 32))
        with pytest.raises(lk.ShapeError):
            lk.launch(dev, lk.binary_collision_kernel, lk.LaunchPlan(extent=16, vvl=4), [bf, bg])
        dev2 = lk.TargetDevice()
        b1 = lk.target_malloc(dev2, lk.FieldDescriptor.create(19, 16))
        b2 = lk.target_malloc(dev2, lk.FieldDescriptor.create(19, 16))
        with pytest.raises(lk.ConfigError):
            lk.launch(dev2, lk.binary_collision_kernel, lk.LaunchPlan(extent=16, vvl=4), [b1, b2])

    def test_noncanonical_cv_rejected(self, lk):
        dev = lk.TargetDevice()
        lk.set_model_constants(dev, lk.D3Q19Model())
        cv = lk.D3Q19Model().cvf[::-1].copy()
        dev.constant_set_double_array("cv", cv, (19, 3))
        b1 = lk.target_malloc(dev, lk.FieldDescriptor.create(19, 16))
        b2 = lk.target_malloc(dev, lk.FieldDescriptor.create(19, 16))
        with pytest.raises(lk.ConfigError):
            lk.launch(dev, lk.binary_collision_kernel, lk.LaunchPlan(extent=16, vvl=4), [b1, b2])

    def test_debug_device_write_tracking(self, lk):
        from paper_1405_6162_b200.verify import run_framework_collision

        f0, g0 = _state(lk, (4, 4, 2), 7)
        plain = run_framework_collision(f0, g0, "cuda", 4, 1)
        tracked = run_framework_collision(f0, g0, "cuda", 4, 1, debug=True)
        assert np.array_equal(plain[0].data, tracked[0].data)
        assert np.array_equal(plain[1].data, tracked[1].data)

    def test_python_kernel_rejected_on_device(self, lk):
        dev = lk.TargetDevice()
        buf = lk.target_malloc(dev, lk.FieldDescriptor.create(1, 8, max_vvl=8))
        with pytest.raises(lk.ConfigError):
            lk.launch(dev, lk.python_kernel("noop", lambda ctx: None),
                      lk.LaunchPlan(extent=8, vvl=8), [buf])


class TestScaleAndMemory:
    def test_scale_bitwise(self, lk, golden):
        from paper_1405_6162_b200.verify import run_framework_scale

        _, small = golden
        d = lk.FieldDescriptor.create(3, 60)
        base = lk.Field(d, small["scale_5x4x3_in"].copy())
        for vvl in (1, 2, 4, 8, 16):
            out = run_framework_scale(base, 0.37, "cuda", vvl)
            assert np.array_equal(out.data, small["scale_5x4x3_out"])

    def test_round_trip_and_zero_init(self, lk):
        dev = lk.TargetDevice()
        desc = lk.FieldDescriptor.create(3, 11)
        buf = lk.target_malloc(dev, desc)
        out = lk.field_create(desc)
        lk.copy_from_target(out, buf)
        assert not out.data.any()
        f = lk.field_create(desc)
        f.data[:] = np.random.default_rng(5).random(desc.nelem)
        lk.copy_to_target(buf, f)
        lk.copy_from_target(out, buf)
        assert np.array_equal(out.data, f.data)
        lk.target_free(buf)
        with pytest.raises(lk.LifecycleError):
            lk.target_free(buf)
        with pytest.raises(lk.LifecycleError):
            lk.copy_to_target(buf, f)

    def test_masked_copies_vs_reference_vectors(self, lk, golden):
        _, small = golden
        dev = lk.TargetDevice()
        k = 0
        while f"mask{k}_flags" in small:
            ncomp, nsites, padded = (int(v) for v in small[f"mask{k}_meta"])
            desc = lk.FieldDescriptor.create(ncomp, nsites, max_vvl=8)
            assert desc.padded_sites == padded
            buf = lk.target_malloc(dev, desc)
            lk.copy_to_target(buf, lk.Field(desc, small[f"mask{k}_init"].copy()))
            flags = small[f"mask{k}_flags"]
            before = dev.counters.elements_packed
            lk.copy_to_target_masked(buf, lk.Field(desc, small[f"mask{k}_host"].copy()),
                                     lk.SiteMask(flags))
            assert dev.counters.elements_packed - before == int(flags.sum()) * ncomp
            out = lk.field_create(desc)
            lk.copy_from_target(out, buf)
            assert np.array_equal(out.data, small[f"mask{k}_out"])
            # and back: masked D2H onto a random host field
            host = lk.Field(desc, np.random.default_rng(k).random(desc.nelem))
            expect = host.data.copy()
            from oracle import oracle as orc
            orc.masked_copy(expect, out.data, ncomp, padded, flags)
            lk.copy_from_target_masked(host, buf, lk.SiteMask(flags))
            assert np.array_equal(host.data, expect)
            lk.target_free(buf)
            k += 1

    def test_isolation_uncopied_reads_zero(self, lk):
        dev = lk.TargetDevice()
        desc = lk.FieldDescriptor.create(19, 64)
        bf, bg = lk.target_malloc(dev, desc), lk.target_malloc(dev, desc)
        host = lk.field_create(desc)
        lk.copy_from_target(host, bf)
        assert not host.data.any()

    def test_in_flight_guard(self, lk):
        # a long launch is still running when the copy is attempted
        from paper_1405_6162_b200.kernels import random_binary_state

        shape = lk.LatticeShape(256, 128, 64)
        f, g = random_binary_state(shape, np.random.default_rng(1))
        dev = lk.TargetDevice()
        lk.set_model_constants(dev, lk.D3Q19Model())
        bf, bg = lk.target_malloc(dev, f.descriptor), lk.target_malloc(dev, g.descriptor)
        lk.copy_to_target(bf, f)
        lk.copy_to_target(bg, g)
        plan = lk.LaunchPlan(extent=f.descriptor.padded_sites, vvl=1)
        for _ in range(40):
            lk.launch(dev, lk.binary_collision_kernel, plan, [bf, bg])
        with pytest.raises((lk.ConcurrencyError, lk.LifecycleError)):
            lk.copy_from_target(f, bf)
            lk.target_free(bf)
        lk.sync_target(dev)
        lk.copy_from_target(f, bf)


class TestBenchApi:
    def test_benchmark_run_and_report(self, lk):
        rows = lk.run_sweep("binary-collision", lk.LatticeShape(32, 32, 32), [1, 2, 4, 8], [1],
                            ["cuda"], iterations=5)
        assert len(rows) == 4 and all(r.sites_per_s > 0 for r in rows)
        lines = lk.report_best(rows)
        assert lines[0].startswith("binary-collision/cuda: best VVL=")
        assert lk.emit_csv(rows).startswith("kernel,backend,nx,ny,nz,vvl,workers,tpb,iters")


class TestEdgeCases:
    def test_ragged_and_tiny_lattices_bitwise(self, lk):
        from oracle import oracle as orc
        from paper_1405_6162_b200.verify import run_framework_collision

        for shape in ((1, 1, 1), (5, 7, 3), (1, 1, 17), (9, 1, 1)):
            f0, g0 = _state(lk, shape, 8)
            n, P = f0.descriptor.nsites, f0.descriptor.padded_sites
            for vvl in (1, 2, 4, 8, 16):
                f1, g1 = run_framework_collision(f0, g0, "cuda", vvl, 1, steps=2)
                rf, rg = f0.data.copy(), g0.data.copy()
                orc.collide(rf, rg, P, n, steps=2)
                assert np.array_equal(f1.data, rf) and np.array_equal(g1.data, rg), (shape, vvl)

    def test_partial_chunk_range(self, lk):
        # a launch over a sub-range of chunks touches exactly those sites
        from paper_1405_6162_b200 import _native as nat
        import ctypes

        f0, g0 = _state(lk, (8, 8, 8), 3)
        P = f0.descriptor.padded_sites
        dev = lk.TargetDevice()
        bf, bg = lk.target_malloc(dev, f0.descriptor), lk.target_malloc(dev, g0.descriptor)
        lk.copy_to_target(bf, f0)
        lk.copy_to_target(bg, g0)
        m = lk.D3Q19Model()
        prm = lk.kernels.collision_params(m.wv, m.cs2, 1.0, 1.0)
        nat.check(nat.lib.ltk_collide(10, 20, 4, 128, bf.ptr, bg.ptr, P, 512, ctypes.byref(prm),
                                      dev.stream))
        lk.sync_target(dev)
        out = lk.field_create(f0.descriptor)
        lk.copy_from_target(out, bf)
        from oracle import oracle as orc
        rf, rg = f0.data.copy(), g0.data.copy()
        orc.lib().orc_collide(orc._p(rf), orc._p(rg), P, 512, orc._p(orc.WV),
                              orc._p(orc.CV.astype(float)), orc.CS2, 1.0, 1.0, 40, 80)
        assert np.array_equal(out.data, rf)

    def test_prepared_parameters_follow_constant_updates(self, lk):
        # launch() reuses the prepared parameter block between identical launches;
        # a constant update between launches (tau_f 1.0 -> 0.8) must reach the
        # kernel, and a launch on other buffers must use those buffers
        from oracle import oracle as orc

        f0, g0 = _state(lk, (8, 8, 8), 11)
        P, n = f0.descriptor.padded_sites, f0.descriptor.nsites
        dev = lk.TargetDevice()
        lk.set_model_constants(dev, lk.D3Q19Model())
        bufs = [lk.target_malloc(dev, f0.descriptor) for _ in range(4)]
        for b, src in zip(bufs, (f0, g0, f0, g0)):
            lk.copy_to_target(b, src)
        plan = lk.LaunchPlan(extent=P, vvl=2)
        lk.launch(dev, lk.binary_collision_kernel, plan, bufs[:2])
        lk.sync_target(dev)
        dev.constant_set_double("tau_f", 0.8)
        lk.launch(dev, lk.binary_collision_kernel, plan, bufs[:2])
        lk.sync_target(dev)
        lk.launch(dev, lk.binary_collision_kernel, plan, bufs[2:])  # same constants, other buffers
        lk.sync_target(dev)
        got = []
        for b in bufs:
            out = lk.field_create(f0.descriptor)
            lk.copy_from_target(out, b)
            got.append(out.data)
        rf, rg = f0.data.copy(), g0.data.copy()
        orc.collide(rf, rg, P, n, tau_f=1.0, tau_g=1.0)
        orc.collide(rf, rg, P, n, tau_f=0.8, tau_g=1.0)
        sf, sg = f0.data.copy(), g0.data.copy()
        orc.collide(sf, sg, P, n, tau_f=0.8, tau_g=1.0)
        assert np.array_equal(got[0], rf) and np.array_equal(got[1], rg)
        assert np.array_equal(got[2], sf) and np.array_equal(got[3], sg)

    def test_nan_input_propagates_like_reference(self, lk):
        from oracle import oracle as orc
        from paper_1405_6162_b200.verify import run_framework_collision

        f0, g0 = _state(lk, (4, 4, 4), 1)
        f0.data[5] = np.nan      # comp 0 of site 5
        g0.data[64 * 3 + 9] = np.inf
        f1, g1 = run_framework_collision(f0, g0, "cuda", 1, 1)
        rf, rg = f0.data.copy(), g0.data.copy()
        orc.collide(rf, rg, 64, 64)
        assert np.array_equal(np.isnan(f1.data), np.isnan(rf))
        fin = np.isfinite(rf)
        assert np.array_equal(f1.data[fin], rf[fin])

    def test_invalid_plans_rejected(self, lk):
        f0, g0 = _state(lk, (4, 4, 4), 1)
        dev = lk.TargetDevice()
        lk.set_model_constants(dev, lk.D3Q19Model())
        bf, bg = lk.target_malloc(dev, f0.descriptor), lk.target_malloc(dev, g0.descriptor)
        with pytest.raises(lk.PlanError):
            lk.launch(dev, lk.binary_collision_kernel, lk.LaunchPlan(extent=128, vvl=2), [bf, bg])
        with pytest.raises(lk.PlanError):  # VVL 32 not compiled
            lk.launch(dev, lk.binary_collision_kernel, lk.LaunchPlan(extent=64, vvl=32), [bf, bg])
        other = lk.TargetDevice()
        with pytest.raises(lk.DeviceError):
            lk.launch(other, lk.binary_collision_kernel, lk.LaunchPlan(extent=64, vvl=2), [bf, bg])


class TestStress:
    def test_repeated_golden_runs_are_stable(self, lk, golden):
        # guards against order-dependent nondeterminism: the 8^3 golden case,
        # 40 times over VVL 1/2 and two TPBs, interleaved with a large launch
        from paper_1405_6162_b200.verify import run_framework_collision

        meta, _ = golden
        case = meta["collision"][0]
        model = lk.D3Q19Model()
        f0, g0 = _state(lk, case["shape"], case["seed"], model)
        big_f, big_g = _state(lk, (128, 128, 64), 2, model)
        for k in range(40):
            vvl, tpb = (1, 2)[k % 2], (128, 256)[(k // 2) % 2]
            f1, g1 = run_framework_collision(f0, g0, "cuda", vvl, 1, steps=case["steps"],
                                             model=model, tpb=tpb)
            assert sha(f1.data) == case["out_f"] and sha(g1.data) == case["out_g"], (k, vvl, tpb)
            if k % 10 == 0:
                run_framework_collision(big_f, big_g, "cuda", 2, 1, steps=1, model=model)


class TestExactDivision:
    """EXACT mode divides by launch constants and by rho through precomputed
    reciprocals (ltk_common.cuh div_rcp, Markstein's theorem).  Checked here
    against the hardware IEEE division on operands spanning the normal
    exponent range, plus signed zeros, infinities and NaN: bitwise equal
    wherever the quotient and the residual stay normal."""

    def test_div_rcp_equals_ieee_division(self, lk):
        from paper_1405_6162_b200 import _native as nat

        rng = np.random.default_rng(20141406)
        n = 4_000_000
        x = rng.uniform(1.0, 2.0, n) * np.exp2(rng.integers(-480, 480, n)) * \
            rng.choice([-1.0, 1.0], n)
        d = rng.uniform(1.0, 2.0, n) * np.exp2(rng.integers(-480, 480, n))
        # the constants EXACT mode divides by, and lattice-scale operands
        consts = np.array([1 / 3, 2 / 3, 2 / 9, 1 / 9, 0.8, 0.9, 1.1, 1.3, 0.51, 1.0])
        d[: n // 4] = rng.choice(consts, n // 4)
        x[: n // 4] = rng.standard_normal(n // 4) * np.exp2(rng.integers(-60, 4, n // 4))
        # rho-like divisors (near 1) with momentum-like numerators
        d[n // 4: n // 2] = 1.0 + 0.2 * rng.random(n // 4)
        x[n // 4: n // 2] = rng.standard_normal(n // 4) * 1e-3
        specials = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-300, -3e-290, 5e300])
        x[-len(specials):] = specials
        d[-len(specials):] = 0.8
        buf = [nat.malloc(8 * n) for _ in range(4)]
        try:
            nat.check(nat.lib.ltk_h2d(buf[0], x.ctypes.data, 8 * n, None))
            nat.check(nat.lib.ltk_h2d(buf[1], d.ctypes.data, 8 * n, None))
            nat.check(nat.lib.ltk_div_selftest(buf[0], buf[1], n, buf[2], buf[3], None))
            got, ref = np.empty(n), np.empty(n)
            nat.check(nat.lib.ltk_d2h(got.ctypes.data, buf[2], 8 * n, None))
            nat.check(nat.lib.ltk_d2h(ref.ctypes.data, buf[3], 8 * n, None))
            nat.check(nat.lib.ltk_stream_sync(None))
        finally:
            for b in buf:
                nat.free(b)
        assert np.array_equal(ref, x / d, equal_nan=True)   # the device IEEE division is numpy's
        nan = np.isnan(ref)
        assert np.array_equal(np.isnan(got), nan)
        same = got[~nan].view(np.uint64) == ref[~nan].view(np.uint64)
        assert same.all(), (x[~nan][~same][:5], d[~nan][~same][:5])


class TestLaunchSequences:
    def test_random_launch_sequences_match_oracle(self, lk):
        # launch() reuses the prepared parameter block while (kernel, plan, buffers,
        # constants) are unchanged: random interleavings of constant updates, plan
        # changes and buffer pairs on one device must still give the oracle's bits
        import os

        from hypothesis import given, settings
        from hypothesis import strategies as st

        from oracle import oracle as orc

        shape = lk.LatticeShape(6, 5, 4)
        f0, g0 = _state(lk, (6, 5, 4), 21)
        P, n = f0.descriptor.padded_sites, f0.descriptor.nsites
        op = st.one_of(
            st.tuples(st.just("tau_f"), st.sampled_from([0.7, 0.8, 1.0, 1.3])),
            st.tuples(st.just("tau_g"), st.sampled_from([0.6, 1.0, 1.7])),
            st.tuples(st.just("launch"), st.integers(0, 1), st.sampled_from([1, 2, 4, 8, 16]),
                      st.sampled_from([32, 64, 128, 256])))

        @settings(max_examples=int(os.environ.get("LTK_HYP_EXAMPLES", "30")), deadline=None)
        @given(ops=st.lists(op, min_size=1, max_size=12))
        def run(ops):
            dev = lk.TargetDevice()
            try:
                lk.set_model_constants(dev, lk.D3Q19Model())
                pairs = []
                for _ in range(2):
                    bf = lk.target_malloc(dev, f0.descriptor)
                    bg = lk.target_malloc(dev, g0.descriptor)
                    lk.copy_to_target(bf, f0)
                    lk.copy_to_target(bg, g0)
                    pairs.append((bf, bg))
                host = [(f0.data.copy(), g0.data.copy()) for _ in range(2)]
                tau = {"tau_f": 1.0, "tau_g": 1.0}
                for o in ops:
                    if o[0] in tau:
                        dev.constant_set_double(o[0], o[1])
                        tau[o[0]] = o[1]
                        continue
                    _, k, vvl, tpb = o
                    plan = lk.LaunchPlan(extent=P, vvl=vvl, tpb=tpb)
                    lk.launch(dev, lk.binary_collision_kernel, plan, list(pairs[k]))
                    lk.sync_target(dev)
                    orc.collide(host[k][0], host[k][1], P, n, tau_f=tau["tau_f"],
                                tau_g=tau["tau_g"])
                for (bf, bg), (hf, hg) in zip(pairs, host):
                    out_f, out_g = lk.field_create(f0.descriptor), lk.field_create(g0.descriptor)
                    lk.copy_from_target(out_f, bf)
                    lk.copy_from_target(out_g, bg)
                    assert np.array_equal(out_f.data, hf) and np.array_equal(out_g.data, hg)
            finally:
                dev.close()

        run()
