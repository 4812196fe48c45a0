"""Multi-slab engine on one B200: the peer transport.

test_engines_in_one_process_*: P engines (slabs) of one process on the same
GPU, attached to each other directly (ltk_fluid_attach_peer_engines) and
stepped alternately from the host; their streams run concurrently, the
kernels store halo images into the neighbour engines' buffers and the
progress counters order the phases -- the code path multi-GPU runs take, with
device pointers instead of IPC mappings.

test_two_process_*: the IPC variant, one process per slab.

Each process owns one z-slab (nranks = 2), exports its buffers with CUDA IPC,
attaches the other process as the slab above and below, and the kernels store
their halo images straight into the neighbour's buffers, ordered by progress
counters.  On one GPU the two contexts time-slice, so this is a correctness
test of the multi-GPU code path (the same path runs on NVLink peers), not a
timing.  The gathered lattice must equal the oracle bitwise.
"""

import os
import socket

import numpy as np
import pytest

from conftest import ROOT, gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shape, steps, physics, q, layout=0):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_1405_6162_b200 as lk
    from paper_1405_6162_b200.kernels import random_binary_state

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = lk.LatticeShape(*shape)
        model = lk.D3Q19Model(tau_f=0.9, tau_g=1.1)
        sim = lk.BinaryFluid(full, model=model, physics=physics, rank=rank, nranks=world,
                             use_graph=False)
        sim.set_layout(layout)
        blob = torch.frombuffer(bytearray(sim.ipc_blob()), dtype=torch.uint8)
        blobs = [torch.zeros_like(blob) for _ in range(world)]
        dist.all_gather(blobs, blob)
        raw = [bytes(b.numpy().tobytes()) for b in blobs]
        sim.attach_peers(raw[(rank + 1) % world], raw[(rank - 1) % world])
        dist.barrier()  # every inbox reset before any neighbour primes it
        f0, g0 = random_binary_state(full, np.random.default_rng(31), model)
        sim.load(f0, g0)
        sim.run(steps)
        f, g = sim.fields(slab_only=True)
        timed_out = sim.peer_timed_out()
        n = f.descriptor.nsites
        mine = torch.from_numpy(np.stack([f.components()[:, :n], g.components()[:, :n]]).copy())
        parts = [torch.zeros_like(mine) for _ in range(world)] if rank == 0 else None
        dist.gather(mine, parts, dst=0)
        sim.close()
        if rank == 0:
            from oracle import oracle as orc

            nx, ny, nz = shape
            nzl = nz // world
            got = [np.concatenate([p.numpy()[k].reshape(19, nx, ny, nzl) for p in parts], axis=3)
                   for k in (0, 1)]
            prm = orc.fluid_params(tau_f=0.9, tau_g=1.1, physics=1 if physics == "binary" else 0)
            P = f0.descriptor.padded_sites
            of, og, _, _ = orc.fluid_step(f0.data, g0.data, shape, P, prm, steps=steps)
            ref = [a.reshape(19, P)[:, :nx * ny * nz].reshape(19, nx, ny, nz) for a in (of, og)]
            ok = all(np.array_equal(a.view(np.uint64), b.view(np.uint64))
                     for a, b in zip(got, ref))
            q.put((bool(ok), bool(timed_out)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


# variant: "plain" (SoA f/g), "vvl2", "row" (the row-blocked f/g layout)
@pytest.mark.parametrize("nslabs", [2, 3, 4])
@pytest.mark.parametrize("physics", ["binary", "passive", "binary-stress"])
@pytest.mark.parametrize("nz,variant", [(12, "plain"), (24, "plain"), (12, "vvl2"), (24, "row")])
def test_engines_in_one_process_bitwise(nslabs, physics, nz, variant):
    import paper_1405_6162_b200 as lk
    from oracle import oracle as orc
    from paper_1405_6162_b200.kernels import random_binary_state

    shape, steps = (32, 8, nz), 4
    full = lk.LatticeShape(*shape)
    model = lk.D3Q19Model(tau_f=0.9, tau_g=1.1)
    sims = [lk.BinaryFluid(full, model=model, physics=physics, rank=r, nranks=nslabs,
                           use_graph=False, vvl=2 if variant == "vvl2" else 1)
            for r in range(nslabs)]
    for sim in sims:
        sim.set_layout(lk.LAYOUT_ROW if variant == "row" else lk.LAYOUT_SOA)
    try:
        for r, sim in enumerate(sims):
            sim.attach_peer_engines(sims[(r + 1) % nslabs], sims[(r - 1) % nslabs])
        # a first state, one step, then a re-load: the halos must be re-primed
        fa, ga = random_binary_state(full, np.random.default_rng(7), model)
        for sim in sims:
            sim.load(fa, ga)
        for sim in sims:
            sim.run(1)
        f0, g0 = random_binary_state(full, np.random.default_rng(31), model)
        for sim in sims:
            sim.load(f0, g0)
        for _ in range(steps):
            for sim in sims:  # interleaved enqueue: every wait has its producer queued
                sim.run(1)
        parts = [sim.fields(slab_only=True) for sim in sims]
        assert not any(sim.peer_timed_out() for sim in sims)
    finally:
        for sim in sims:
            sim.close()
    nx, ny, nz = shape
    nzl = nz // nslabs
    got = [np.concatenate([p[k].components()[:, :nx * ny * nzl].reshape(19, nx, ny, nzl)
                           for p in parts], axis=3) for k in (0, 1)]
    prm = orc.fluid_params(tau_f=0.9, tau_g=1.1,
                           physics={"passive": 0, "binary": 1, "binary-stress": 2}[physics])
    P = f0.descriptor.padded_sites
    of, og, _, _ = orc.fluid_step(f0.data, g0.data, shape, P, prm, steps=steps)
    ref = [a.reshape(19, P)[:, :nx * ny * nz].reshape(19, nx, ny, nz) for a in (of, og)]
    for a, b in zip(got, ref):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("physics,layout", [("binary", 0), ("passive", 0), ("binary", 1)])
def test_two_process_peer_slabs_bitwise(physics, layout):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    shape, steps = (16, 8, 12), 3
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shape, steps, physics, q, layout))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    codes = [p.exitcode for p in procs]
    for p in procs:
        if p.is_alive():
            p.kill()
    assert codes == [0, 0], codes
    ok, timed_out = q.get(timeout=5)
    assert not timed_out
    assert ok


def test_engines_in_one_process_random_bitwise():
    """Hypothesis over the peer transport: slab count, slab depth, plane shape,
    physics, layout; the gathered lattice bitwise vs the oracle.
    LTK_HYP_EXAMPLES raises the example count (default 15)."""
    from hypothesis import given, settings
    from hypothesis import strategies as st

    import paper_1405_6162_b200 as lk
    from oracle import oracle as orc
    from paper_1405_6162_b200.kernels import random_binary_state

    n = int(os.environ.get("LTK_HYP_EXAMPLES", "15"))

    @settings(max_examples=n, deadline=None)
    @given(nslabs=st.integers(2, 4), nzl=st.integers(2, 6),
           nx=st.sampled_from([2, 6, 16, 32]), ny=st.sampled_from([1, 3, 8, 16]),
           physics=st.sampled_from(["passive", "binary", "binary-stress"]),
           row=st.booleans(), steps=st.integers(1, 3), seed=st.integers(0, 10 ** 6))
    def check(nslabs, nzl, nx, ny, physics, row, steps, seed):
        seen.append((nslabs, row, nzl))
        shape = (nx, ny, nslabs * nzl)
        full = lk.LatticeShape(*shape)
        model = lk.D3Q19Model(tau_f=0.9, tau_g=1.1)
        sims = [lk.BinaryFluid(full, model=model, physics=physics, rank=r, nranks=nslabs,
                               use_graph=False) for r in range(nslabs)]
        try:
            for sim in sims:
                sim.set_layout(lk.LAYOUT_ROW if row else lk.LAYOUT_SOA)
            for r, sim in enumerate(sims):
                sim.attach_peer_engines(sims[(r + 1) % nslabs], sims[(r - 1) % nslabs])
            f0, g0 = random_binary_state(full, np.random.default_rng(seed), model)
            for sim in sims:
                sim.load(f0, g0)
            for _ in range(steps):
                for sim in sims:
                    sim.run(1)
            parts = [sim.fields(slab_only=True) for sim in sims]
            assert not any(sim.peer_timed_out() for sim in sims)
        finally:
            for sim in sims:
                sim.close()
        nz = nslabs * nzl
        got = [np.concatenate([p[k].components()[:, :nx * ny * nzl].reshape(19, nx, ny, nzl)
                               for p in parts], axis=3) for k in (0, 1)]
        prm = orc.fluid_params(tau_f=0.9, tau_g=1.1,
                               physics={"passive": 0, "binary": 1, "binary-stress": 2}[physics])
        P = f0.descriptor.padded_sites
        of, og, _, _ = orc.fluid_step(f0.data, g0.data, shape, P, prm, steps=steps)
        ref = [a.reshape(19, P)[:, :nx * ny * nz].reshape(19, nx, ny, nz) for a in (of, og)]
        for a, b in zip(got, ref):
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), (shape, nslabs, physics)

    seen = []
    check()
    print(f"random peer-slab parity: {len(seen)} examples, "
          f"{sum(1 for c in seen if c[0] >= 3)} with 3-4 slabs, "
          f"{sum(1 for c in seen if c[1])} row-blocked, {sum(1 for c in seen if c[2] == 2)} "
          f"with 2-plane slabs")


def test_stalled_neighbour_raises():
    """A progress wait that times out (a neighbour slab stalled) must not go on
    silently with stale halos: sync() raises DeviceError on that engine and the
    engine refuses further steps.  The timeout is injected (the real budget is
    ~8 s of spinning)."""
    import paper_1405_6162_b200 as lk
    from paper_1405_6162_b200.kernels import random_binary_state

    full = lk.LatticeShape(16, 8, 8)
    sims = [lk.BinaryFluid(full, rank=r, nranks=2, use_graph=False) for r in range(2)]
    try:
        for r, sim in enumerate(sims):
            sim.attach_peer_engines(sims[1 - r], sims[1 - r])
        f0, g0 = random_binary_state(full, np.random.default_rng(3))
        for sim in sims:
            sim.load(f0, g0)
        sims[0].inject_peer_timeout()
        for sim in sims:
            sim.run(1)
        with pytest.raises(lk.DeviceError, match="timed out"):
            sims[0].sync()
        assert sims[0].peer_timed_out()
        with pytest.raises(lk.DeviceError):
            sims[0].run(1)
    finally:
        for sim in sims:
            sim.close()


@pytest.mark.parametrize("transport", ["peer"])
def test_bench_eight_ranks_bitwise(tmp_path, transport):
    """`python bench.py --gpus 8` without a launcher: it
    spawns 8 ranks itself, they share this test box's one GPU over the peer
    transport, the line reports n_gpus 8 with one record per rank, and the
    state dumped after the timed steps equals the oracle bitwise."""
    import json
    import subprocess
    import sys

    from oracle import oracle as orc
    from paper_1405_6162_b200.kernels import random_binary_state
    import paper_1405_6162_b200 as lk

    nx, ny, nzl, world, seed = 16, 16, 4, 8, 77
    prefix = str(tmp_path / "state")
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, "bench.py", "--gpus", str(world), "--shape",
                          f"{nx}x{ny}x{nzl}", "--steps", "3", "--warmup", "3", "--no-e2e",
                          "--no-cpu-baseline", "--no-config1", "--seed", str(seed),
                          "--transport", transport, "--dump", prefix],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == world and len(line["ranks"]) == world
    assert sorted(r["rank"] for r in line["ranks"]) == list(range(world))
    assert line["config"]["halo_transport"] == transport and not line["peer_wait_timeout"]
    assert line["dump"]["steps"] == 6

    # the same initial state (bench.py: slab r from rng(seed + r)), whole lattice
    model = lk.D3Q19Model()
    full = lk.LatticeShape(nx, ny, nzl * world)
    from paper_1405_6162_b200.lattice import FieldDescriptor, field_create

    desc = FieldDescriptor.create(19, full.nsites)
    f0, g0 = field_create(desc), field_create(desc)
    for r in range(world):
        fs, gs = random_binary_state(lk.LatticeShape(nx, ny, nzl), np.random.default_rng(seed + r),
                                     model)
        for dst, src in ((f0, fs), (g0, gs)):
            for i in range(19):
                d = dst.component(i).reshape(nx, ny, nzl * world)
                d[:, :, r * nzl:(r + 1) * nzl] = src.component(i).reshape(nx, ny, nzl)
    prm = orc.fluid_params(tau_f=1.0, tau_g=1.0, physics=1)
    of, og, _, _ = orc.fluid_step(f0.data, g0.data, (nx, ny, nzl * world), desc.padded_sites,
                                  prm, steps=6)
    from paper_1405_6162_b200 import io as lio

    fd, shape = lio.read_slab(prefix + ".f", 0, nzl * world)
    gd, _ = lio.read_slab(prefix + ".g", 0, nzl * world)
    assert shape == full
    n = full.nsites
    for got, ref in ((fd, of), (gd, og)):
        assert np.array_equal(got.data.reshape(19, -1)[:, :n],
                              ref.reshape(19, -1)[:, :n])
