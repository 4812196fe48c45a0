"""HBM read-only vs copy bandwidth on the box (torch kernels, CUDA events):
the ceiling for read-dominated kernels such as k_phi (152 B read : 8 B written)."""
import torch

n = 19 * 256 ** 3  # one g state, 2.55 GB
x = torch.rand(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def best(fn, nbytes, reps=10):
    fn()
    torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        t.append(s.elapsed_time(e))
    return nbytes / min(t) / 1e6


print("read  (sum) %.0f GB/s" % best(lambda: x.sum(), 8 * n))
print("copy        %.0f GB/s" % best(lambda: y.copy_(x), 16 * n))
print("write (fill)%.0f GB/s" % best(lambda: y.fill_(1.0), 8 * n))
