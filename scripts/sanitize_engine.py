"""Small engine runs for compute-sanitizer (memcheck / racecheck): every layout,
force form, VVL 2, the peer transport between in-process slabs, ragged plane
counts for k_mu_tile (nzl not a multiple of its 8-plane blocks) and the plain
mu kernel (ny % 8 != 0).  Prints one line per case; exits 1 on a
result that differs from the single-slab SoA run.

    compute-sanitizer --tool memcheck python scripts/sanitize_engine.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1405_6162_b200 as lk  # noqa: E402
from paper_1405_6162_b200.kernels import random_binary_state  # noqa: E402


def run(shape, layout, physics="binary", vvl=1, nslabs=1, steps=3):
    full = lk.LatticeShape(*shape)
    model = lk.D3Q19Model(tau_f=0.9, tau_g=1.1)
    f0, g0 = random_binary_state(full, np.random.default_rng(5), model)
    sims = [lk.BinaryFluid(full, model=model, physics=physics, vvl=vvl, rank=r, nranks=nslabs,
                           use_graph=False) for r in range(nslabs)]
    try:
        for s in sims:
            s.set_layout(layout)
        if nslabs > 1:
            for r, s in enumerate(sims):
                s.attach_peer_engines(sims[(r + 1) % nslabs], sims[(r - 1) % nslabs])
        for s in sims:
            s.load(f0, g0)
        for _ in range(steps):
            for s in sims:
                s.run(1)
        parts = [s.fields(slab_only=nslabs > 1) for s in sims]
        tot = sum(s.totals() for s in sims)
    finally:
        for s in sims:
            s.close()
    nx, ny, nz = shape
    nzl = nz // nslabs
    if nslabs == 1:
        return parts[0][0].data, parts[0][1].data, tot
    got = [np.concatenate([p[k].components()[:, :nx * ny * nzl].reshape(19, nx, ny, nzl)
                           for p in parts], axis=3) for k in (0, 1)]
    return got[0], got[1], tot


def main():
    bad = 0
    cases = [
        dict(shape=(32, 8, 11), physics="binary"),
        dict(shape=(32, 8, 11), physics="binary-stress"),
        dict(shape=(32, 8, 11), physics="passive"),
        dict(shape=(32, 8, 12), vvl=2),
        dict(shape=(32, 6, 12)),
        dict(shape=(64, 16, 5), physics="binary-stress"),
        dict(shape=(16, 6, 12), nslabs=2),
        dict(shape=(16, 6, 12), nslabs=3, physics="binary-stress"),
    ]
    for c in cases:
        ref_c = dict(c)
        nsl = ref_c.pop("nslabs", 1)
        ref = run(layout=lk.LAYOUT_SOA, **ref_c)
        for layout in (lk.LAYOUT_SOA, lk.LAYOUT_ROW):
            got = run(layout=layout, **c)
            shape = c["shape"]
            if nsl > 1:  # compare in (comp, x, y, z) form
                n = shape[0] * shape[1] * shape[2]
                ref_cmp = [a.reshape(19, -1)[:, :n].reshape(19, *shape) for a in ref[:2]]
            else:
                ref_cmp = ref[:2]
            ok = all(np.array_equal(np.asarray(a), np.asarray(b)) for a, b in zip(got[:2], ref_cmp))
            print(c, "layout", layout, "ok" if ok else "MISMATCH", flush=True)
            bad += not ok
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
