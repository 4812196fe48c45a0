"""Timing of one full step's kernels at 256^3 (FAST) -- k_mu TMA vs before."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1405_6162_b200 as lk
from paper_1405_6162_b200 import _native as nat
from paper_1405_6162_b200.kernels import random_binary_state
shape = lk.LatticeShape(256, 256, 256)
f0, g0 = random_binary_state(shape, np.random.default_rng(1234))
with lk.BinaryFluid(shape, mode=lk.MODE_FAST, use_graph=False) as sim:
    sim.load(f0, g0); sim.run(3); sim.sync()
    sim.profile(True); sim.run(30); sim.sync(); prof = sim.profile(False)
    print("per step ms: phi %.3f mu %.3f cs %.3f total %.3f" % tuple(p / 30 for p in prof))
