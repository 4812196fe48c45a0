"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes tests/golden/reference_golden.json (sha256 of input/output states for
lattices up to 128^3) and tests/golden/reference_small.npz (full arrays for
tiny lattices).  Every vector comes from the reference's own public API:
random_binary_state / equilibrium_binary_state (kernels.py:216-243) for inputs
and verify.run_framework_collision (verify.py:31-51, i.e. the numba
_collision_range, kernels.py:89-125) for outputs.  These files are what the
oracle (oracle/) and the CUDA path are pinned against; nothing on the GPU box
reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

import latkit  # the reference package (PYTHONPATH above)
from latkit import D3Q19Model, LatticeShape, SiteMask, TargetDevice
from latkit.kernels import (bgk_relax, equilibrium, equilibrium_binary_state, moments,
                            random_binary_state, random_vector_field)
from latkit.memory import copy_from_target, copy_to_target, copy_to_target_masked, target_malloc
from latkit.lattice import FieldDescriptor, field_create
from latkit.verify import run_framework_collision, run_framework_scale

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


# (nx, ny, nz, seed, steps, tau_f, tau_g, vvl) -- the first two are the
# reference's own bitwise tests (test_kernels.py:174-185, test_acceptance.py:82-91)
COLLISION_CASES = [
    (8, 8, 8, 5, 2, 1.0, 1.0, 8),
    (8, 8, 8, 20140708, 5, 1.0, 1.0, 8),
    (16, 16, 16, 20140707, 1, 1.0, 1.0, 4),
    (3, 3, 3, 6, 1, 1.0, 1.0, 8),
    (5, 4, 3, 11, 3, 0.8, 1.3, 4),
    (32, 32, 32, 1234, 3, 0.8, 1.3, 8),
    (32, 32, 32, 1234, 10, 1.0, 1.0, 2),
    (128, 128, 128, 1234, 1, 0.8, 1.0, 8),
]


def main() -> None:
    golden = {"reference": "latkit " + getattr(latkit, "__version__", "?"),
              "collision": [], "scale": [], "equilibrium_state": {}}
    small = {}

    for nx, ny, nz, seed, steps, tf, tg, vvl in COLLISION_CASES:
        shape = LatticeShape(nx, ny, nz)
        model = D3Q19Model(tau_f=tf, tau_g=tg)
        f0, g0 = random_binary_state(shape, np.random.default_rng(seed), model)
        f1, g1 = run_framework_collision(f0, g0, "reference", vvl, 1, steps=steps, model=model)
        entry = dict(shape=[nx, ny, nz], seed=seed, steps=steps, tau_f=tf, tau_g=tg,
                     padded=f0.descriptor.padded_sites,
                     in_f=sha(f0.data), in_g=sha(g0.data),
                     out_f=sha(f1.data), out_g=sha(g1.data))
        golden["collision"].append(entry)
        if shape.nsites <= 64:
            key = f"coll_{nx}x{ny}x{nz}_s{seed}"
            small[key + "_in_f"], small[key + "_in_g"] = f0.data, g0.data
            small[key + "_out_f"], small[key + "_out_g"] = f1.data, g1.data
        print("collision", entry["shape"], "steps", steps, file=sys.stderr)

    # scale kernel (kernels.py:79-86) via the reference framework
    for nx, ny, nz, seed, a in ((5, 4, 3, 3, 0.37), (16, 16, 16, 20140707, 0.37)):
        shape = LatticeShape(nx, ny, nz)
        base = random_vector_field(shape, np.random.default_rng(seed))
        out = run_framework_scale(base, a, "reference", 4, 1)
        golden["scale"].append(dict(shape=[nx, ny, nz], seed=seed, a=a,
                                    padded=base.descriptor.padded_sites,
                                    in_=sha(base.data), out=sha(out.data)))
        if shape.nsites <= 64:
            small[f"scale_{nx}x{ny}x{nz}_in"] = base.data
            small[f"scale_{nx}x{ny}x{nz}_out"] = out.data

    # equilibrium fixed point (verify.py:154-165)
    model = D3Q19Model()
    feq, geq = equilibrium_binary_state(LatticeShape(4, 4, 4), 1.0, (0.02, -0.01, 0.03), 0.3, model)
    f1, g1 = run_framework_collision(feq, geq, "reference", 4, 1, model=model)
    small["eqstate_in_f"], small["eqstate_in_g"] = feq.data, geq.data
    small["eqstate_out_f"], small["eqstate_out_g"] = f1.data, g1.data

    # site operations (kernels.py:29-73)
    rho, u = moments(model.wv, model)
    small["site_moments_wv"] = np.array([rho, *u])
    small["site_equilibrium"] = equilibrium(1.2, (0.03, -0.05, 0.02), model)
    rng = np.random.default_rng(0)
    fsite = model.wv * (1.0 + 0.1 * rng.random(19))
    r, uu = moments(fsite, model)
    small["site_relax_in"] = fsite
    small["site_relax_out"] = bgk_relax(fsite, equilibrium(r, uu, model), 0.8)

    # masked transfers (memory.py:277-315) on the emulated discrete target
    rng = np.random.default_rng(20140710)
    dev = TargetDevice(backend="emulated")
    for k in range(12):
        nsites = int(rng.integers(1, 65))
        ncomp = int(rng.choice([1, 3, 19]))
        desc = FieldDescriptor.create(ncomp, nsites, max_vvl=8)
        flags = rng.random(nsites) < rng.random()
        host = field_create(desc)
        host.data[:] = rng.random(desc.nelem)
        init = field_create(desc)
        init.data[:] = rng.random(desc.nelem)
        buf = target_malloc(dev, desc)
        copy_to_target(buf, init)
        copy_to_target_masked(buf, host, SiteMask(flags))
        out = field_create(desc)
        copy_from_target(out, buf)
        small[f"mask{k}_flags"] = flags
        small[f"mask{k}_meta"] = np.array([ncomp, nsites, desc.padded_sites])
        small[f"mask{k}_host"] = host.data
        small[f"mask{k}_init"] = init.data
        small[f"mask{k}_out"] = out.data

    with open(os.path.join(HERE, "reference_golden.json"), "w") as fh:
        json.dump(golden, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "reference_small.npz"), **small)
    print("wrote", len(golden["collision"]), "collision cases,", len(small), "arrays",
          file=sys.stderr)


if __name__ == "__main__":
    main()
