"""Multi-slab overhead on ONE B200 (proxy for the scaling design): P engines
of 256x256x(256/P) joined by the peer transport, stepped together, vs one
engine of 256^3; and the NCCL slab path (self-communicator) vs the local path."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1405_6162_b200 as lk
from paper_1405_6162_b200 import _native as nat
from paper_1405_6162_b200.kernels import random_binary_state

MODE = lk.MODE_FAST if "--fast" in sys.argv else lk.MODE_EXACT  # bench default: EXACT
full = lk.LatticeShape(256, 256, 256)
f0, g0 = random_binary_state(full, np.random.default_rng(1234))
res = {}
for P in (1, 2, 4, 8):
    sims = [lk.BinaryFluid(full, mode=MODE, rank=r, nranks=P, use_graph=(P == 1))
            for r in range(P)]
    if P > 1:
        for r, sim in enumerate(sims):
            sim.attach_peer_engines(sims[(r + 1) % P], sims[(r - 1) % P])
    for sim in sims:
        sim.load(f0, g0)
    for _ in range(3):
        for sim in sims:
            sim.run(1)
    for sim in sims:
        sim.sync()
    s, e = nat.event_create(True), nat.event_create(True)
    nat.lib.ltk_event_record(s, sims[0].stream)
    # the other streams start after s
    for sim in sims[1:]:
        nat.lib.ltk_stream_wait_event(sim.stream, s)
    steps = 20
    for _ in range(steps):
        for sim in sims:
            sim.run(1)
    ends = []
    for sim in sims:
        ev = nat.event_create(True)
        nat.lib.ltk_event_record(ev, sim.stream)
        ends.append(ev)
    for sim in sims:
        sim.sync()
    ms = max(nat.elapsed_ms(s, ev) for ev in ends) / steps
    res[f"peer P={P}"] = ms
    print(f"peer transport, {P} slabs of 256x256x{256 // P} on one GPU: {ms:.3f} ms/step "
          f"{full.nsites / ms / 1e6:.2f} GLUPS, timeouts={[x.peer_timed_out() for x in sims]}",
          flush=True)
    for sim in sims:
        sim.close()

if lk.nccl_available():
    sim = lk.BinaryFluid(full, mode=MODE, use_graph=False)
    sim.attach_nccl(lk.nccl_unique_id())
    sim.load(f0, g0); sim.run(3); sim.sync()
    s, e = nat.event_create(True), nat.event_create(True)
    nat.lib.ltk_event_record(s, sim.stream); sim.run(20); nat.lib.ltk_event_record(e, sim.stream); sim.sync()
    ms = nat.elapsed_ms(s, e) / 20
    print(f"NCCL slab path (self communicator, P=1) 256^3: {ms:.3f} ms/step {full.nsites / ms / 1e6:.2f} GLUPS", flush=True)
    sim.close()
