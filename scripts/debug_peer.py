"""Two processes on one GPU: inspect peer-transport halos after load / 1 step."""
import os, sys, socket
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def worker(rank, world, port):
    import ctypes
    import torch, torch.distributed as dist
    import paper_1405_6162_b200 as lk
    from paper_1405_6162_b200 import _native as nat
    from paper_1405_6162_b200.kernels import random_binary_state
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shape = lk.LatticeShape(16, 8, 12)
    sim = lk.BinaryFluid(shape, rank=rank, nranks=world, use_graph=False)
    blob = torch.frombuffer(bytearray(sim.ipc_blob()), dtype=torch.uint8)
    blobs = [torch.zeros_like(blob) for _ in range(world)]
    dist.all_gather(blobs, blob)
    raw = [bytes(b.numpy().tobytes()) for b in blobs]
    sim.attach_peers(raw[(rank + 1) % world], raw[(rank - 1) % world])
    dist.barrier()
    f0, g0 = random_binary_state(shape, np.random.default_rng(31))
    sim.load(f0, g0)
    nat.check(nat.lib.ltk_stream_sync(sim.stream))
    dist.barrier()
    ptrs = [ctypes.c_void_p() for _ in range(4)]
    nat.lib.ltk_fluid_buffers(sim.handle, *[ctypes.byref(p) for p in ptrs])
    cs, PL, nzl = sim.slab.cstride, 16 * 8, sim.nzl
    f = np.empty(19 * cs)
    nat.check(nat.lib.ltk_d2h(f.ctypes.data, ptrs[0].value, f.nbytes, None)); nat.lib.ltk_stream_sync(None)
    f = f.reshape(19, cs)[:, :(nzl + 2) * PL].reshape(19, nzl + 2, PL)
    print(f"rank {rank} after load: halo0 comp5 mean {f[5,0].mean():.4f} (own top comp5 {f[5,nzl].mean():.4f}) "
          f"halo_top comp6 mean {f[6,nzl+1].mean():.4f} (own bottom comp6 {f[6,1].mean():.4f}) inbox-wait...", flush=True)
    sim.run(1)
    try:
        sim.sync()
        print(f"rank {rank} step 1 ok, timeout={sim.peer_timed_out()}", flush=True)
    except Exception as e:
        print(f"rank {rank} step 1 error {e}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=worker, args=(r, 2, port)) for r in range(2)]
    [p.start() for p in ps]; [p.join(120) for p in ps]
    print("exit", [p.exitcode for p in ps])
