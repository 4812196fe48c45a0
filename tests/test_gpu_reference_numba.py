"""The device collision against the reference's OWN code at BASELINE sizes.

The golden vectors (tests/golden/) pin the collision on small lattices.  Here
the unmodified reference package installed for the bench's reference arm
(baseline/_ref, `pip install --target`) runs its numba
`_collision_range` through its own launch API on the host cores, and the
B200 path must agree bit for bit at configs[1]'s 128^3 (and on a ragged
lattice whose padding both must leave untouched).  Skipped where the
reference install is absent; nothing here reads /root/reference.
"""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ref(tmp_path_factory):
    if not os.path.isdir(os.path.join(REF, "latkit")):
        pytest.skip("reference not installed in baseline/_ref")
    # the reference's numba kernels use cache=True: keep their cache out of the tree
    os.environ.setdefault("NUMBA_CACHE_DIR", str(tmp_path_factory.mktemp("numba")))
    sys.path.insert(0, REF)
    try:
        import latkit
        import latkit.kernels
        import latkit.verify
    except Exception as exc:  # noqa: BLE001
        pytest.skip(f"reference latkit not importable: {exc}")
    return latkit


@pytest.fixture(scope="module")
def lk():
    import paper_1405_6162_b200 as lk

    return lk


@pytest.mark.parametrize("shape,vvl,taus,steps", [
    ((128, 128, 128), 1, (1.0, 1.0), 2),
    ((128, 128, 128), 2, (0.8, 1.1), 2),
    ((33, 17, 9), 8, (0.9, 0.7), 3),
])
def test_collision_bitwise_vs_reference_numba(ref, lk, shape, vvl, taus, steps):
    from paper_1405_6162_b200.kernels import random_binary_state
    from paper_1405_6162_b200.verify import run_framework_collision

    workers = os.cpu_count() or 1
    rmodel = ref.D3Q19Model(tau_f=taus[0], tau_g=taus[1])
    rf0, rg0 = ref.kernels.random_binary_state(ref.LatticeShape(*shape),
                                               np.random.default_rng(20140707), rmodel)
    rf, rg = ref.verify.run_framework_collision(rf0, rg0, "threaded", vvl, workers, steps=steps,
                                                model=rmodel)
    model = lk.D3Q19Model(tau_f=taus[0], tau_g=taus[1])
    f0, g0 = random_binary_state(lk.LatticeShape(*shape), np.random.default_rng(20140707), model)
    assert np.array_equal(f0.data, rf0.data) and np.array_equal(g0.data, rg0.data)  # same inputs
    f1, g1 = run_framework_collision(f0, g0, "threaded", vvl, workers, steps=steps, model=model)
    assert np.array_equal(f1.data.view(np.uint64), rf.data.view(np.uint64))
    assert np.array_equal(g1.data.view(np.uint64), rg.data.view(np.uint64))


def test_scale_bitwise_vs_reference_numba(ref, lk):
    from paper_1405_6162_b200.kernels import random_vector_field
    from paper_1405_6162_b200.verify import run_framework_scale

    shape = (128, 128, 128)
    rv = ref.kernels.random_vector_field(ref.LatticeShape(*shape), np.random.default_rng(7))
    want = ref.verify.run_framework_scale(rv, 0.37, "threaded", 4, os.cpu_count() or 1)
    v = random_vector_field(lk.LatticeShape(*shape), np.random.default_rng(7))
    got = run_framework_scale(v, 0.37, "threaded", 4, 1)
    assert np.array_equal(got.data.view(np.uint64), want.data.view(np.uint64))


def test_passive_step_equals_reference_collision_after_streaming(ref, lk):
    # the engine's full step in the passive limit (no force, no chemical potential) is
    # the reference collision applied to the pulled (streamed) state: three steps at 64^3
    # against numpy streaming + the reference's own numba collision, bitwise
    from paper_1405_6162_b200.kernels import random_binary_state

    shape = (64, 64, 64)
    nx, ny, nz = shape
    n = nx * ny * nz
    model = lk.D3Q19Model(tau_f=0.9, tau_g=1.2)
    f0, g0 = random_binary_state(lk.LatticeShape(*shape), np.random.default_rng(11), model)
    with lk.BinaryFluid(lk.LatticeShape(*shape), model=model, physics="passive") as sim:
        sim.load(f0, g0)
        sim.run(3)
        f1, g1 = sim.fields()
    P = f0.descriptor.padded_sites
    cv = np.asarray(model.cv, dtype=int)

    def stream(a):  # f_i(x) <- f_i(x - c_i), host order s = (x*ny + y)*nz + z, periodic
        out = a.copy().reshape(19, P)
        for i in range(19):
            v = out[i, :n].reshape(nx, ny, nz)
            out[i, :n] = np.roll(v, tuple(cv[i]), axis=(0, 1, 2)).ravel()
        return out.ravel()

    rmodel = ref.D3Q19Model(tau_f=0.9, tau_g=1.2)
    rdesc = ref.FieldDescriptor.create(19, n)
    rf = ref.Field(rdesc, f0.data.copy())
    rg = ref.Field(rdesc, g0.data.copy())
    for _ in range(3):
        rf = ref.Field(rdesc, stream(rf.data))
        rg = ref.Field(rdesc, stream(rg.data))
        rf, rg = ref.verify.run_framework_collision(rf, rg, "threaded", 1, os.cpu_count() or 1,
                                                    model=rmodel)
    assert np.array_equal(f1.data.view(np.uint64), rf.data.view(np.uint64))
    assert np.array_equal(g1.data.view(np.uint64), rg.data.view(np.uint64))
