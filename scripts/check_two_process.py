"""Two CUDA processes on one GPU: H2D round trip and slab scatter per process (the
cross-process check behind tests/test_gpu_peer.py::test_two_process_*)."""
import os, sys, socket, ctypes, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def worker(rank, world, port, delay):
    import torch, torch.distributed as dist
    import paper_1405_6162_b200 as lk
    from paper_1405_6162_b200 import _native as nat
    from paper_1405_6162_b200.kernels import random_binary_state
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if delay and rank == 1:
        time.sleep(3)
    shape = lk.LatticeShape(16, 8, 12)
    f0, g0 = random_binary_state(shape, np.random.default_rng(31))
    sim = lk.BinaryFluid(shape, rank=rank, nranks=world, use_graph=False)
    nb = f0.descriptor.nbytes
    st = nat.malloc(2 * nb)
    rc1 = nat.lib.ltk_h2d(st, f0.data.ctypes.data, nb, sim.stream)
    rc2 = nat.lib.ltk_stream_sync(sim.stream)
    back = np.empty_like(f0.data)
    rc3 = nat.lib.ltk_d2h(back.ctypes.data, st, nb, sim.stream); nat.lib.ltk_stream_sync(sim.stream)
    print(rank, "h2d roundtrip ok", np.array_equal(back, f0.data), rc1, rc2, rc3, nat.last_error(), flush=True)
    slab = sim.slab
    rc4 = nat.lib.ltk_fluid_scatter(ctypes.byref(slab), st, f0.descriptor.padded_sites, 12, sim.z0, 19,
                                    ctypes.c_void_p(0) if False else None, sim.stream) if False else 0
    ptrs = [ctypes.c_void_p() for _ in range(4)]
    nat.lib.ltk_fluid_buffers(sim.handle, *[ctypes.byref(p) for p in ptrs])
    rc5 = nat.lib.ltk_fluid_scatter(ctypes.byref(slab), st, f0.descriptor.padded_sites, 12, sim.z0, 19,
                                    ptrs[0].value, sim.stream)
    rc6 = nat.lib.ltk_stream_sync(sim.stream)
    cs, PL, nzl = slab.cstride, 128, sim.nzl
    f = np.empty(19 * cs)
    rc7 = nat.lib.ltk_d2h(f.ctypes.data, ptrs[0].value, f.nbytes, sim.stream); nat.lib.ltk_stream_sync(sim.stream)
    f = f.reshape(19, cs)[:, :(nzl + 2) * PL].reshape(19, nzl + 2, PL)
    print(rank, "scatter rc", rc5, rc6, rc7, "own mean", f[:, 1:nzl + 1].mean(), nat.last_error(), flush=True)
    dev = ctypes.c_int(-1); nat.lib.ltk_get_device(ctypes.byref(dev))
    print(rank, "device", dev.value, "z0", sim.z0, "nzl", nzl, "cstride", cs, flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    for delay in (False, True):
        print("==== delay", delay, flush=True)
        s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
        ctx = mp.get_context("spawn")
        ps = [ctx.Process(target=worker, args=(r, 2, port, delay)) for r in range(2)]
        [p.start() for p in ps]; [p.join(120) for p in ps]
        print("exit", [p.exitcode for p in ps], flush=True)
