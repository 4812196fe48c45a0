import os, sys, socket, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def read_own(sim, nat):
    ptrs = [ctypes.c_void_p() for _ in range(4)]
    nat.lib.ltk_fluid_buffers(sim.handle, *[ctypes.byref(p) for p in ptrs])
    cs, PL, nzl = sim.slab.cstride, 16 * 8, sim.nzl
    f = np.empty(19 * cs)
    nat.check(nat.lib.ltk_d2h(f.ctypes.data, ptrs[0].value, f.nbytes, None)); nat.lib.ltk_stream_sync(None)
    f = f.reshape(19, cs)[:, :(nzl + 2) * PL].reshape(19, nzl + 2, PL)
    return f[5, nzl].mean(), f[6, 1].mean(), f[5, 0].mean(), f[6, nzl + 1].mean(), hex(ptrs[0].value)


def worker(rank, world, port, attach):
    import torch, torch.distributed as dist
    import paper_1405_6162_b200 as lk
    from paper_1405_6162_b200 import _native as nat
    from paper_1405_6162_b200.kernels import random_binary_state
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shape = lk.LatticeShape(16, 8, 12)
    sim = lk.BinaryFluid(shape, rank=rank, nranks=world, use_graph=False)
    print(rank, "fresh", read_own(sim, nat), flush=True)
    blob = sim.ipc_blob()
    import struct
    offs = struct.unpack("<7Q", blob[7 * 64:7 * 64 + 56])
    print(rank, "offsets", offs, flush=True)
    t = torch.frombuffer(bytearray(blob), dtype=torch.uint8)
    blobs = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(blobs, t)
    raw = [bytes(b.numpy().tobytes()) for b in blobs]
    if attach:
        sim.attach_peers(raw[(rank + 1) % world], raw[(rank - 1) % world])
        print(rank, "after attach", read_own(sim, nat), flush=True)
    dist.barrier()
    f0, g0 = random_binary_state(shape, np.random.default_rng(31))
    sim.load(f0, g0)
    nat.check(nat.lib.ltk_stream_sync(sim.stream))
    print(rank, "after load", read_own(sim, nat), flush=True)
    dist.barrier()
    print(rank, "after both loads", read_own(sim, nat), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    for attach in (False, True):
        print("==== attach", attach, flush=True)
        s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
        ctx = mp.get_context("spawn")
        ps = [ctx.Process(target=worker, args=(r, 2, port, attach)) for r in range(2)]
        [p.start() for p in ps]; [p.join(120) for p in ps]
        print("exit", [p.exitcode for p in ps], flush=True)
