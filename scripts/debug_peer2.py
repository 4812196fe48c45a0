import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1405_6162_b200 as lk
from paper_1405_6162_b200 import _native as nat
from paper_1405_6162_b200.kernels import random_binary_state
shape = lk.LatticeShape(16, 8, 12)
f0, g0 = random_binary_state(shape, np.random.default_rng(31))
for nranks, rank in ((1, 0), (2, 0), (2, 1)):
    sim = lk.BinaryFluid(shape, rank=rank, nranks=nranks, use_graph=False)
    if nranks == 2:
        b = sim.ipc_blob()
        print("blob head", b[:16].hex(), flush=True)
    sim.load(f0, g0)
    nat.check(nat.lib.ltk_stream_sync(sim.stream))
    ptrs = [ctypes.c_void_p() for _ in range(4)]
    nat.lib.ltk_fluid_buffers(sim.handle, *[ctypes.byref(p) for p in ptrs])
    cs, PL, nzl = sim.slab.cstride, 16 * 8, sim.nzl
    f = np.empty(19 * cs)
    nat.check(nat.lib.ltk_d2h(f.ctypes.data, ptrs[0].value, f.nbytes, None)); nat.lib.ltk_stream_sync(None)
    f = f.reshape(19, cs)[:, :(nzl + 2) * PL].reshape(19, nzl + 2, PL)
    print(nranks, rank, "own top comp5", f[5, nzl].mean(), "own bottom comp6", f[6, 1].mean(), "ptr", hex(ptrs[0].value), flush=True)
    ff, gg = sim.fields(slab_only=(nranks == 2))
    print("fields mean", ff.data.mean())
    sim.close()
