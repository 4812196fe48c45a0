"""PCIe throughput on the box: H2D / D2H / both, 1..4 streams, pinned 2.55 GB buffers."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1405_6162_b200 import _native as nat
from paper_1405_6162_b200.memory import pinned_empty

n = 19 * 256 ** 3
nb = 8 * n
h_in, h_out = pinned_empty(n), pinned_empty(n)
h_in[:] = 1.0
d_a, d_b = nat.malloc(nb), nat.malloc(nb)
streams = [nat.stream_create() for _ in range(8)]
L = nat.lib


def timed(fn):
    s, e = nat.event_create(True), nat.event_create(True)
    fn()  # warm
    for st in streams:
        L.ltk_stream_sync(st)
    L.ltk_event_record(s, streams[0])
    for st in streams[1:]:
        L.ltk_stream_wait_event(st, s)
    fn()
    for st in streams[1:]:
        ev = nat.event_create(); L.ltk_event_record(ev, st); L.ltk_stream_wait_event(streams[0], ev)
    L.ltk_event_record(e, streams[0])
    L.ltk_event_sync(e)
    return nat.elapsed_ms(s, e)


for k in (1, 2, 4):
    chunk = nb // k

    def h2d():
        for j in range(k):
            L.ltk_h2d(d_a + j * chunk, h_in.ctypes.data + j * chunk, chunk, streams[j])

    def d2h():
        for j in range(k):
            L.ltk_d2h(h_out.ctypes.data + j * chunk, d_b + j * chunk, chunk, streams[4 + j])

    def both():
        h2d(); d2h()

    t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
    print(f"streams/direction={k}: H2D {nb / t1 / 1e6:.1f} GB/s  D2H {nb / t2 / 1e6:.1f} GB/s  "
          f"both {2 * nb / t3 / 1e6:.1f} GB/s total ({t3:.1f} ms for 2 x {nb / 1e9:.2f} GB)", flush=True)
