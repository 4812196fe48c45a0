"""TEST INFRASTRUCTURE: the engine's NCCL transport with P ranks on one GPU.

Loads the NCCL stand-in (nccl_shim.cpp, SONAME libnccl.so.2) before libltk.so
dlopens "libnccl.so.2", so ltk_fluid_attach_nccl / exchange() run their real
code -- face packing in either f/g layout, the fixed send order and mirrored
receives, the comm stream overlapped with the interior planes, unpacking --
with P engines of this process as the ranks, each stepped from its own host
thread.  Prints one JSON line per case: the gathered lattice vs a single-slab
run of the same state, bitwise.  Not importable from the product; run by
tests/test_gpu_nccl_shim.py in a subprocess that never imports torch (torch
would load the real libnccl.so.2).
"""
import ctypes
import json
import os
import sys
import threading

shim = sys.argv[1]
ctypes.CDLL(shim, mode=ctypes.RTLD_GLOBAL)  # before libltk.so's dlopen("libnccl.so.2")
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1405_6162_b200 as lk  # noqa: E402
from paper_1405_6162_b200.kernels import random_binary_state  # noqa: E402

assert "torch" not in sys.modules
steps = 4
for P, shape, physics, layout in [(2, (16, 12, 8), "binary", lk.LAYOUT_ROW),
                                  (3, (16, 12, 9), "binary", lk.LAYOUT_ROW),
                                  (4, (32, 8, 16), "binary", lk.LAYOUT_SOA),
                                  (2, (16, 12, 8), "binary-stress", lk.LAYOUT_ROW),
                                  (3, (16, 12, 6), "passive", lk.LAYOUT_SOA),
                                  (4, (64, 32, 32), "binary", lk.LAYOUT_ROW)]:
    full = lk.LatticeShape(*shape)
    model = lk.D3Q19Model(tau_f=0.9, tau_g=1.1)
    f0, g0 = random_binary_state(full, np.random.default_rng(17), model)
    with lk.BinaryFluid(full, model=model, physics=physics) as one:
        one.set_layout(layout)
        one.load(f0, g0)
        one.run(steps)
        rf, rg = one.fields()
    uid = lk.nccl_unique_id()
    sims = [lk.BinaryFluid(full, model=model, physics=physics, rank=r, nranks=P, use_graph=False)
            for r in range(P)]
    for s in sims:
        s.set_layout(layout)
    for s in sims:
        s.attach_nccl(uid)
    for s in sims:
        s.load(f0, g0)
    errs = []

    def drive(s):
        try:
            s.run(steps)
            s.sync()
        except Exception as exc:  # noqa: BLE001
            errs.append(repr(exc))

    th = [threading.Thread(target=drive, args=(s,)) for s in sims]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    hung = any(t.is_alive() for t in th)
    ok = not hung and not errs
    if ok:
        nx, ny, nz = shape
        nzl = nz // P
        n = full.nsites
        parts = [s.fields(slab_only=True) for s in sims]
        for k, ref in ((0, rf), (1, rg)):
            got = np.concatenate([p[k].components()[:, :nx * ny * nzl].reshape(19, nx, ny, nzl)
                                  for p in parts], axis=3)
            want = ref.components()[:, :n].reshape(19, nx, ny, nz)
            ok = ok and np.array_equal(got.view(np.uint64), want.view(np.uint64))
    for s in sims:
        if not hung:
            s.close()
    print(json.dumps({"P": P, "shape": shape, "physics": physics, "layout": layout,
                      "bitwise_equal_single_slab": bool(ok), "errors": errs, "hung": hung}),
          flush=True)
    if hung:
        os._exit(3)
