"""Drive a few fused steps at 256^3 (for ncu captures)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1405_6162_b200 as lk
from paper_1405_6162_b200.kernels import random_binary_state
shape = lk.LatticeShape(256, 256, 256)
f0, g0 = random_binary_state(shape, np.random.default_rng(1234))
with lk.BinaryFluid(shape, use_graph=False) as sim:
    sim.set_step(lk.STEP_FUSED if (len(sys.argv) < 2 or sys.argv[1] == "fused") else lk.STEP_SPLIT)
    sim.load(f0, g0)
    sim.run(3)
    sim.sync()
print("done")
