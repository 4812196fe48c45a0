"""Locate EXACT-mode VVL=2 mismatches vs the oracle (debug helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1405_6162_b200 as lk
from paper_1405_6162_b200.kernels import random_binary_state
from paper_1405_6162_b200.verify import run_framework_collision
from oracle import oracle as orc

for shape, seed in (((8, 8, 8), 5), ((16, 16, 16), 20140707)):
    for steps in (1, 2):
        for vvl in (1, 2, 4):
            for tpb in (32, 128, 256):
                m = lk.D3Q19Model()
                f0, g0 = random_binary_state(lk.LatticeShape(*shape), np.random.default_rng(seed), m)
                f1, g1 = run_framework_collision(f0, g0, "cuda", vvl, 1, steps=steps, model=m, tpb=tpb)
                rf, rg = f0.data.copy(), g0.data.copy()
                orc.collide(rf, rg, f0.descriptor.padded_sites, f0.descriptor.nsites, steps=steps)
                bad = np.flatnonzero(f1.data.view(np.uint64) != rf.view(np.uint64))
                badg = np.flatnonzero(g1.data.view(np.uint64) != rg.view(np.uint64))
                P = f0.descriptor.padded_sites
                info = ""
                if bad.size:
                    s = bad % P
                    d = (f1.data.view(np.int64)[bad] - rf.view(np.int64)[bad])
                    info = f"sites {np.unique(s)[:8]} comps {np.unique(bad // P)[:8]} ulps {np.unique(d)[:5]}"
                print(shape, steps, "vvl", vvl, "tpb", tpb, "bad f", bad.size, "bad g", badg.size, info)
