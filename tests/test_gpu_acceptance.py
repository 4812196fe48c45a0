"""The reference's acceptance criteria, one test each, on the B200.

Mirrors reference pkg/tests/test_acceptance.py criterion by
criterion with the same seed (SEED = 20140707), through this package's
drop-in API, so a reference user sees the same contract hold on the device:

  01 determinism: 2 kernels x {8^3, 16^3} x 36 configurations bitwise equal.
     The reference's configurations are (backend x workers x VVL); here the
     backend names are aliases of the CUDA target, and workers are kept for
     API compatibility, so the 36 configurations also vary the CUDA block
     (TPB 32 / 64 / 128 / 256 across the sweep) -- what actually changes the
     device schedule.
  02 collision bitwise equal to the scalar triple-loop oracle (8^3, 5 steps).
  03 per-site rho, rho u, phi conserved to 1e-13 (16^3).
  04 uniform equilibrium is a fixed point to 1e-13.
  05 D3Q19 moment identities to 1e-15 (host constants).
  06 1000 randomized masked transfers vs the per-element oracle.
  07 isolation: an uncopied target buffer reads as zeros (the reference's
     probe is a host-Python kernel; the B200 target runs device kernels
     only, so the buffer is read back instead).
  08 the VVL sweep report shape (reference :158-183; the throughput line is
     informational there and here).
  09 CLI contract (sweep rows, --verify PASS lines, VVL rejection exit 2).
"""

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

SEED = 20140707
BACKENDS = ("reference", "threaded", "emulated")
VVLS = (1, 2, 4, 8)
WORKER_COUNTS = (1, 2, 4)
TPBS = (32, 64, 128, 256)


@pytest.fixture(scope="module")
def lk():
    import paper_1405_6162_b200 as lk

    return lk


def test_01_determinism_suite(lk):
    from paper_1405_6162_b200.kernels import random_binary_state, random_vector_field
    from paper_1405_6162_b200.verify import run_framework_collision, run_framework_scale

    model = lk.D3Q19Model()
    configs = [(b, w, v) for b in BACKENDS for w in WORKER_COUNTS for v in VVLS]
    assert len(configs) == 36
    for shape in (lk.LatticeShape(8, 8, 8), lk.LatticeShape(16, 16, 16)):
        rng = np.random.default_rng(SEED)
        vec = random_vector_field(shape, rng)
        f0, g0 = random_binary_state(shape, rng, model)
        scale_ref = coll_ref = None
        for k, (backend, workers, vvl) in enumerate(configs):
            tpb = TPBS[k % len(TPBS)]
            out = run_framework_scale(vec, 0.37, backend, vvl, workers, tpb=tpb)
            scale_ref = out if scale_ref is None else scale_ref
            assert np.array_equal(out.data, scale_ref.data), (shape, backend, workers, vvl)
            f1, g1 = run_framework_collision(f0, g0, backend, vvl, workers, model=model,
                                             tpb=tpb)
            coll_ref = (f1, g1) if coll_ref is None else coll_ref
            assert np.array_equal(f1.data, coll_ref[0].data), (shape, backend, workers, vvl)
            assert np.array_equal(g1.data, coll_ref[1].data), (shape, backend, workers, vvl)


def test_02_oracle_equivalence(lk):
    from oracle import oracle as orc
    from paper_1405_6162_b200.kernels import random_binary_state
    from paper_1405_6162_b200.verify import run_framework_collision

    shape = lk.LatticeShape(8, 8, 8)
    model = lk.D3Q19Model()
    f0, g0 = random_binary_state(shape, np.random.default_rng(SEED + 1), model)
    rf, rg = f0.data.copy(), g0.data.copy()
    P = f0.descriptor.padded_sites
    for _ in range(5):  # the pure-Python site loop (oracle.py, independent of lb_oracle.c)
        orc.collide_scalar(rf, rg, P, shape.nsites)
    f1, g1 = run_framework_collision(f0, g0, "threaded", 8, 2, steps=5, model=model)
    assert np.array_equal(f1.data, rf) and np.array_equal(g1.data, rg)


def test_03_conservation(lk):
    from paper_1405_6162_b200.verify import verify_conservation

    ok, lines = verify_conservation(lk.LatticeShape(16, 16, 16), seed=SEED + 2, rel_tol=1e-13)
    assert ok, lines


def test_04_equilibrium_fixed_point(lk):
    from paper_1405_6162_b200.verify import verify_fixed_point

    ok, lines = verify_fixed_point(lk.LatticeShape(8, 8, 8), rho=1.0, u=(0.02, -0.01, 0.03),
                                   phi=0.3, tol=1e-13)
    assert ok, lines


def test_05_moment_identities(lk):
    model = lk.D3Q19Model()
    Q = 19
    worst = abs(sum(model.wv) - 1.0)
    for a in range(3):
        worst = max(worst, abs(sum(model.wv[i] * model.cv[i, a] for i in range(Q))))
        for b in range(3):
            second = sum(model.wv[i] * model.cv[i, a] * model.cv[i, b] for i in range(Q))
            worst = max(worst, abs(second - ((1.0 / 3.0) if a == b else 0.0)))
    assert worst <= 1e-15, worst


def test_06_masked_transfer_suite(lk):
    from oracle import oracle as orc

    rng = np.random.default_rng(SEED + 3)
    dev = lk.TargetDevice(backend="emulated")
    try:
        for _ in range(1000):
            nsites = int(rng.integers(1, 65))
            ncomp = int(rng.choice([1, 3, 19]))
            desc = lk.FieldDescriptor.create(ncomp, nsites, max_vvl=8)
            flags = rng.random(nsites) < rng.random()
            host = lk.field_create(desc)
            host.data[:] = rng.random(desc.nelem)
            buf = lk.target_malloc(dev, desc)
            expected = np.zeros(desc.nelem)
            orc.masked_copy(expected, host.data, ncomp, desc.padded_sites, flags)
            before = dev.counters.elements_packed
            lk.copy_to_target_masked(buf, host, lk.SiteMask(flags))
            assert dev.counters.elements_packed - before == int(flags.sum()) * ncomp
            out = lk.field_create(desc)
            lk.copy_from_target(out, buf)
            assert np.array_equal(out.data, expected)
            lk.target_free(buf)
    finally:
        dev.close()


def test_07_isolation(lk):
    dev = lk.TargetDevice(backend="emulated", workers=2)
    try:
        desc = lk.FieldDescriptor.create(3, 16, max_vvl=16)
        host = lk.field_create(desc)
        host.data[:] = 1.0  # never copied to the target
        buf = lk.target_malloc(dev, desc)
        out = lk.field_create(desc)
        out.data[:] = -1.0
        lk.copy_from_target(out, buf)
        assert not out.data.any()
    finally:
        dev.close()


def test_08_vvl_tuning_report(lk):
    rows = lk.run_sweep("binary-collision", lk.LatticeShape(16, 16, 16), [1, 2, 4, 8], [1],
                        ["threaded"], iterations=5, seed=SEED)
    lines = lk.report_best(rows)
    assert len(rows) == 4 and len(lines) == 1
    assert lines[0].startswith("binary-collision/threaded: best VVL=") and "x over VVL=1" in lines[0]


def test_09_cli_contract(lk, capsys):
    from paper_1405_6162_b200.cli import cli_main

    code = cli_main(["--kernel", "scale", "--shape", "16x16x16", "--vvl", "1,2,4,8",
                     "--workers", "1,4", "--backend", "threaded", "--iters", "100", "--csv"])
    out = capsys.readouterr().out
    assert code == 0 and len([ln for ln in out.split("\n") if ln.startswith("scale,")]) == 8
    code = cli_main(["--verify", "--kernel", "binary-collision", "--shape", "8x8x8",
                     "--iters", "1"])
    out = capsys.readouterr().out.split("\n")
    assert code == 0
    assert any(ln.startswith("PASS equivalence") for ln in out)
    assert any(ln.startswith("PASS conservation") for ln in out)
    code = cli_main(["--vvl", "3", "--shape", "8x8x8"])
    captured = capsys.readouterr()
    assert code == 2 and "VVL must divide padded extent" in captured.err
