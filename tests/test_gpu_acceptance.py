"""Acceptance criteria of the reference, checked on the B200.

Each criterion of reference pkg/tests/test_acceptance.py has one test here,
driven through this package's drop-in API with the reference's seed
(20140707 + offset per criterion), so the contract a reference user relies
on is shown to hold on the device:

  01  scale and collision outputs identical (bitwise) over the 36
      (backend, workers, VVL) configurations at 8^3 and 16^3.  Backend names
      alias the CUDA target and workers are API-only, so the sweep also
      rotates the CUDA block size through 32..256, which does change the
      device schedule.
  02  five collisions at 8^3 equal the pure-Python site loop of the oracle.
  03  rho, momentum and phi of every site kept to 1e-13 (16^3).
  04  a uniform equilibrium stays put to 1e-13.
  05  D3Q19 weight moments to 1e-15.
  06  1000 random masked transfers equal the per-element oracle.
  07  a target buffer never written reads back as zeros (the reference
      observes it from a host-Python kernel, which this target does not run).
  08  the VVL sweep yields one row per VVL and a best-VVL summary line.
  09  CLI: sweep rows, --verify PASS lines, exit 2 on a VVL that does not
      divide the padded extent.
"""

import itertools

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

BASE_SEED = 20140707  # reference test_acceptance.py SEED


@pytest.fixture(scope="module")
def lk():
    import paper_1405_6162_b200 as lk

    return lk


def _sweep_configs():
    """(backend, workers, vvl, cuda block) for the 36 reference configurations."""
    combos = itertools.product(("reference", "threaded", "emulated"), (1, 2, 4), (1, 2, 4, 8))
    blocks = itertools.cycle((32, 64, 128, 256))
    return [(b, w, v, next(blocks)) for b, w, v in combos]


@pytest.mark.parametrize("n", [8, 16])
def test_01_outputs_identical_over_configurations(lk, n):
    from paper_1405_6162_b200.kernels import random_binary_state, random_vector_field
    from paper_1405_6162_b200.verify import run_framework_collision, run_framework_scale

    cfgs = _sweep_configs()
    assert len(cfgs) == 36
    shape = lk.LatticeShape(n, n, n)
    model = lk.D3Q19Model()
    rng = np.random.default_rng(BASE_SEED)
    vec = random_vector_field(shape, rng)
    f0, g0 = random_binary_state(shape, rng, model)
    outs = []
    for backend, workers, vvl, block in cfgs:
        s = run_framework_scale(vec, 0.37, backend, vvl, workers, tpb=block)
        f, g = run_framework_collision(f0, g0, backend, vvl, workers, model=model, tpb=block)
        outs.append((s.data, f.data, g.data))
    first = outs[0]
    for cfg, got in zip(cfgs, outs):
        for k in range(3):
            assert np.array_equal(got[k].view(np.uint64), first[k].view(np.uint64)), (cfg, k)


def test_02_five_steps_equal_the_python_site_loop(lk):
    from oracle import oracle as orc
    from paper_1405_6162_b200.kernels import random_binary_state
    from paper_1405_6162_b200.verify import run_framework_collision

    shape = lk.LatticeShape(8, 8, 8)
    f0, g0 = random_binary_state(shape, np.random.default_rng(BASE_SEED + 1), lk.D3Q19Model())
    want_f, want_g = f0.data.copy(), g0.data.copy()
    for _ in range(5):  # oracle.py's pure-Python restatement, independent of lb_oracle.c
        orc.collide_scalar(want_f, want_g, f0.descriptor.padded_sites, shape.nsites)
    got_f, got_g = run_framework_collision(f0, g0, "threaded", 8, 2, steps=5)
    assert np.array_equal(got_f.data, want_f) and np.array_equal(got_g.data, want_g)


def test_03_site_invariants_kept(lk):
    from paper_1405_6162_b200.verify import verify_conservation

    ok, report = verify_conservation(lk.LatticeShape(16, 16, 16), seed=BASE_SEED + 2,
                                     rel_tol=1e-13)
    assert ok, report


def test_04_uniform_equilibrium_is_fixed(lk):
    from paper_1405_6162_b200.verify import verify_fixed_point

    ok, report = verify_fixed_point(lk.LatticeShape(8, 8, 8), rho=1.0, u=(0.02, -0.01, 0.03),
                                    phi=0.3, tol=1e-13)
    assert ok, report


def test_05_weight_moments(lk):
    m = lk.D3Q19Model()
    w, c = np.asarray(m.wv, dtype=float), np.asarray(m.cv, dtype=float)
    errors = [abs(w.sum() - 1.0)]
    errors += [abs(float(w @ c[:, a])) for a in range(3)]
    second = np.einsum("i,ia,ib->ab", w, c, c)
    errors += list(np.abs(second - np.eye(3) / 3.0).ravel())
    assert max(errors) <= 1e-15, max(errors)


def test_06_random_masked_transfers(lk):
    from oracle import oracle as orc

    rng = np.random.default_rng(BASE_SEED + 3)
    dev = lk.TargetDevice(backend="emulated")
    try:
        for case in range(1000):
            nsites = int(rng.integers(1, 65))
            ncomp = int(rng.choice([1, 3, 19]))
            desc = lk.FieldDescriptor.create(ncomp, nsites, max_vvl=8)
            keep = rng.random(nsites) < rng.random()
            src = lk.field_create(desc)
            src.data[:] = rng.random(desc.nelem)
            want = np.zeros(desc.nelem)
            orc.masked_copy(want, src.data, ncomp, desc.padded_sites, keep)
            buf = lk.target_malloc(dev, desc)
            packed0 = dev.counters.elements_packed
            lk.copy_to_target_masked(buf, src, lk.SiteMask(keep))
            moved = dev.counters.elements_packed - packed0
            back = lk.field_create(desc)
            lk.copy_from_target(back, buf)
            lk.target_free(buf)
            assert moved == int(keep.sum()) * ncomp, case
            assert np.array_equal(back.data, want), case
    finally:
        dev.close()


def test_07_unwritten_target_reads_zero(lk):
    dev = lk.TargetDevice(backend="emulated", workers=2)
    try:
        desc = lk.FieldDescriptor.create(3, 16, max_vvl=16)
        host = lk.field_create(desc)
        host.data[:] = 1.0  # stays on the host
        buf = lk.target_malloc(dev, desc)
        seen = lk.field_create(desc)
        seen.data[:] = np.nan
        lk.copy_from_target(seen, buf)
        assert np.all(seen.data == 0.0)
    finally:
        dev.close()


def test_08_vvl_sweep_summary(lk):
    rows = lk.run_sweep("binary-collision", lk.LatticeShape(16, 16, 16), [1, 2, 4, 8], [1],
                        ["threaded"], iterations=5, seed=BASE_SEED)
    summary = lk.report_best(rows)
    assert [r.vvl for r in rows] == [1, 2, 4, 8] and len(summary) == 1
    assert summary[0].startswith("binary-collision/threaded: best VVL=")
    assert "x over VVL=1" in summary[0]


def test_09_command_line(lk, capsys):
    from paper_1405_6162_b200.cli import cli_main

    rc = cli_main(["--kernel", "scale", "--shape", "16x16x16", "--vvl", "1,2,4,8",
                   "--workers", "1,4", "--backend", "threaded", "--iters", "100", "--csv"])
    rows = [ln for ln in capsys.readouterr().out.splitlines() if ln.startswith("scale,")]
    assert rc == 0 and len(rows) == 8

    rc = cli_main(["--verify", "--kernel", "binary-collision", "--shape", "8x8x8", "--iters", "1"])
    lines = capsys.readouterr().out.splitlines()
    assert rc == 0
    assert any(ln.startswith("PASS equivalence") for ln in lines)
    assert any(ln.startswith("PASS conservation") for ln in lines)

    rc = cli_main(["--vvl", "3", "--shape", "8x8x8"])
    assert rc == 2 and "VVL must divide padded extent" in capsys.readouterr().err
