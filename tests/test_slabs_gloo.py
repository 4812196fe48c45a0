"""Multi-rank z-slab decomposition on CPU: world_size 2 (and 3) over gloo.

Each rank owns nz/P planes plus halo planes (one per face for f, g, phi; two
for mu, which the filtered potential force reads at z +- 2), exchanges
exactly the halo ops of slabs.halo_schedule (the order the C++ engine issues
its NCCL send/recv), and steps its slab with the numpy restatement of the
timestep.
The gathered lattice must equal the single-domain oracle bitwise: this pins
the decomposition, the crossing-component sets and the send/recv matching
that the GPU engine relies on, with no GPU and no cluster.
"""

import os
import socket

import numpy as np
import pytest

from conftest import ROOT

SHAPE = (6, 5, 12)
STEPS = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _exchange(dist, torch, arrays, ops, rank):
    """Run one schedule group; arrays: dict kind -> ndarray (comp?, zs, y, x)."""
    reqs, recvs = [], []
    count = {}
    for op in ops:
        key = (op.op, op.peer)
        tag = count.get(key, 0)
        count[key] = tag + 1
        a = arrays[op.kind]
        if op.kind == "mu":          # two planes per face
            view = a[op.plane:op.plane + 2]
        else:
            view = a[op.comp, op.plane] if a.ndim == 4 else a[op.plane]
        if op.op == "send":
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(view)), op.peer, tag=tag))
        else:
            buf = torch.empty(view.shape, dtype=torch.float64)
            reqs.append(dist.irecv(buf, op.peer, tag=tag))
            recvs.append((view, buf))
    for r in reqs:
        r.wait()
    for view, buf in recvs:
        view[...] = buf.numpy()


def _worker(rank, world, port, out_q):
    import torch
    import torch.distributed as dist

    import sys
    sys.path.insert(0, ROOT)
    from oracle import oracle as orc
    from paper_1405_6162_b200.slabs import halo_schedule, slab_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, ny, nz = SHAPE
    n = nx * ny * nz
    P = -(-n // 16) * 16
    f0, g0 = orc.random_binary_state(n, P, 17)
    prm = orc.fluid_params(tau_f=0.85, tau_g=1.2, physics=1)
    z0, nzl = slab_bounds(nz, rank, world)

    def to_slab(a):
        full = a.reshape(19, P)[:, :n].reshape(19, nx, ny, nz).transpose(0, 3, 2, 1)
        s = np.zeros((19, nzl + 2, ny, nx))
        s[:, 1:nzl + 1] = full[:, z0:z0 + nzl]
        return s

    f, g = to_slab(f0), to_slab(g0)
    phi = np.zeros((nzl + 2, ny, nx))
    mu = np.zeros((nzl + 4, ny, nx))      # mu layout: zs = z + 2
    cv = orc.CV
    for _ in range(STEPS):
        _exchange(dist, torch, {"f": f, "g": g}, halo_schedule("fg", rank, world, nzl), rank)
        fs = np.stack([np.roll(f[i, 1 - cv[i, 2]:nzl + 1 - cv[i, 2]], (cv[i, 1], cv[i, 0]), (1, 2))
                       for i in range(19)])
        gs = np.stack([np.roll(g[i, 1 - cv[i, 2]:nzl + 1 - cv[i, 2]], (cv[i, 1], cv[i, 0]), (1, 2))
                       for i in range(19)])
        ph = np.zeros((nzl, ny, nx))
        for i in range(19):
            ph = ph + gs[i]
        phi[1:nzl + 1] = ph
        _exchange(dist, torch, {"phi": phi}, halo_schedule("phi", rank, world, nzl), rank)
        nb = [np.roll(ph, -1, 2), np.roll(ph, 1, 2), np.roll(ph, -1, 1), np.roll(ph, 1, 1),
              phi[2:nzl + 2], phi[0:nzl]]
        mu[2:nzl + 2] = orc.mu_numpy(ph, nb, prm)
        _exchange(dist, torch, {"mu": mu}, halo_schedule("mu", rank, world, nzl), rank)
        m = mu[2:nzl + 2]
        # filtered potential force (orc_potential_force op order); in z, h on
        # planes -1..nzl from the phi halos and the two mu halo planes per face
        force = []
        for ax in (2, 1):   # x, y (in-plane, periodic)
            h = -(ph * ((np.roll(m, -1, ax) - np.roll(m, 1, ax)) * 0.5))
            force.append(((np.roll(h, 1, ax) + np.roll(h, -1, ax)) + (h + h)) * 0.25)
        hz = -(phi[0:nzl + 2] * ((mu[2:nzl + 4] - mu[0:nzl + 2]) * 0.5))
        force.append(((hz[0:nzl] + hz[2:nzl + 2]) + (hz[1:nzl + 1] + hz[1:nzl + 1])) * 0.25)
        fo, go = orc.collide_streamed_numpy(fs.reshape(19, -1), gs.reshape(19, -1), m.ravel(),
                                            [c.ravel() for c in force], prm)
        f = np.zeros_like(f)
        g = np.zeros_like(g)
        f[:, 1:nzl + 1] = fo.reshape(19, nzl, ny, nx)
        g[:, 1:nzl + 1] = go.reshape(19, nzl, ny, nx)
    # gather owned planes on rank 0 and compare with the global oracle
    mine = torch.from_numpy(np.ascontiguousarray(np.stack([f[:, 1:nzl + 1], g[:, 1:nzl + 1]])))
    parts = [torch.empty_like(mine) for _ in range(world)] if rank == 0 else None
    dist.gather(mine, parts, dst=0)
    if rank == 0:
        full = np.concatenate([p.numpy() for p in parts], axis=2)  # (2, 19, nz, ny, nx)
        of, og, _, _ = orc.fluid_step(f0, g0, SHAPE, P, prm, steps=STEPS)
        ref = [a.reshape(19, P)[:, :n].reshape(19, nx, ny, nz).transpose(0, 3, 2, 1)
               for a in (of, og)]
        ok = (np.array_equal(full[0].view(np.uint64), ref[0].view(np.uint64)) and
              np.array_equal(full[1].view(np.uint64), ref[1].view(np.uint64)))
        out_q.put(bool(ok))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_slabs_bitwise_equal_global(world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) is True
