"""Full-duplex PCIe with write-combined vs cached pinned H2D sources (4 streams
per direction, 2 x 2.55 GB each way), CUDA events; cuda-python for the
allocation flags.  Experiment for the e2e leg of bench.py."""
import ctypes
import sys

sys.path.insert(0, ".")
from cuda.bindings import runtime as rt  # noqa: E402

from paper_1405_6162_b200 import _native as nat  # noqa: E402

nb = 19 * 256 ** 3 * 8
L = nat.lib


def halloc(flags):
    err, p = rt.cudaHostAlloc(nb, flags)
    assert err == rt.cudaError_t.cudaSuccess, err
    ctypes.memset(p, 1, nb)
    return p


src = {"cached": [halloc(0), halloc(0)], "wc": [halloc(rt.cudaHostAllocWriteCombined)] * 1}
src["wc"].append(halloc(rt.cudaHostAllocWriteCombined))
dst = [halloc(0), halloc(0)]
dev_in = [nat.malloc(nb), nat.malloc(nb)]
dev_out = [nat.malloc(nb), nat.malloc(nb)]
S = 4
hs = [nat.stream_create() for _ in range(S)]
ds = [nat.stream_create() for _ in range(S)]
ch = nb // 2


def duplex(kind):
    j = 0
    for c in range(2):
        for part in range(2):
            L.ltk_h2d(dev_in[c] + part * ch, src[kind][c] + part * ch, ch, hs[j % S])
            L.ltk_d2h(dst[c] + part * ch, dev_out[c] + part * ch, ch, ds[j % S])
            j += 1


def timed(kind, reps=3):
    best = 1e9
    for _ in range(reps):
        a, b = nat.event_create(True), nat.event_create(True)
        for s in hs + ds:
            L.ltk_stream_sync(s)
        L.ltk_event_record(a, hs[0])
        for s in hs[1:] + ds:
            L.ltk_stream_wait_event(s, a)
        duplex(kind)
        for s in hs[1:] + ds:
            e = nat.event_create()
            L.ltk_event_record(e, s)
            L.ltk_stream_wait_event(hs[0], e)
        L.ltk_event_record(b, hs[0])
        L.ltk_event_sync(b)
        best = min(best, nat.elapsed_ms(a, b))
    return best


for kind in ("cached", "wc", "cached", "wc"):
    ms = timed(kind)
    print(f"{kind:7s} duplex 2 x {2 * nb / 1e9:.2f} GB: {ms:.1f} ms = {4 * nb / ms / 1e6:.1f} GB/s total",
          flush=True)
