"""z-slab decomposition: geometry, the halo-exchange schedule, and a
one-device multi-slab stepper.

The production multi-GPU path is the C++ engine (csrc/fluid.cu): one slab
per rank, halo planes stored by the producing kernels into the neighbours
over NVLink (peer transport) or NCCL send/recv (`exchange`), overlapped with
the interior planes.  This module states the same
decomposition in Python so that it can be checked without several GPUs:

* `slab_bounds`, `halo_schedule` -- the ownership and the ordered
  send/recv list the engine issues (faces up first, then down; receives
  mirror that order so per-peer matching holds for P = 1, 2 and > 2);
* `VirtualSlabs` -- P slabs on ONE device, each stepped with the C-ABI
  kernels (ltk_fluid_phi / _mu / _collide_stream) and halos moved with
  ltk_fluid_pack_face / unpack_face and plane copies; bitwise equal to the
  single-slab engine (tests/test_gpu_fluid.py);
* tests/test_slabs_gloo.py runs the schedule across 2 gloo processes on CPU.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import ConfigError, ShapeError, SingularStateError
from .lattice import Field, FieldDescriptor, LatticeShape, field_create
from .model import CZ_DOWN, CZ_UP, Q


def slab_bounds(nz: int, rank: int, nranks: int) -> tuple[int, int]:
    """(z0, nzl): rank owns global planes [z0, z0 + nzl)."""
    if nranks < 1 or not 0 <= rank < nranks:
        raise ShapeError(f"bad rank {rank} of {nranks}")
    if nz % nranks:
        raise ShapeError(f"nz {nz} not divisible by {nranks} ranks")
    nzl = nz // nranks
    return rank * nzl, nzl


def neighbours(rank: int, nranks: int) -> tuple[int, int]:
    """(up, down) = ranks owning the planes above / below this slab (periodic)."""
    return (rank + 1) % nranks, (rank - 1) % nranks


@dataclass(frozen=True)
class HaloOp:
    """One point-to-point transfer of a halo plane.

    kind: "fg" (distribution component `comp` of dist "f" or "g"), "phi", "mu".
    plane: storage plane index zs (owned z = zs - 1; 0 and nzl + 1 are halos).
    """

    op: str        # "send" | "recv"
    peer: int
    kind: str      # "f", "g", "phi", "mu"
    comp: int      # distribution component (or 0 for phi/mu)
    plane: int


def halo_schedule(kind: str, rank: int, nranks: int, nzl: int) -> list[HaloOp]:
    """Ordered ops of one exchange group, exactly as the engine issues them.

    kind "fg": crossing components of f then g (the engine packs them into
    one contiguous face per direction, in this order); "phi": one plane each
    way; "mu": two planes each way (mu layout, zs = z + 2).
    fg / phi sends: top owned plane (zs = nzl) up, bottom owned plane (zs = 1)
    down; receives: from down into zs = 0, from up into zs = nzl + 1.
    mu sends: planes zs = nzl, nzl + 1 up and zs = 2, 3 down; receives from
    down into zs = 0, 1 and from up into zs = nzl + 2, nzl + 3 (`plane` is the
    first of the pair).
    """
    up, down = neighbours(rank, nranks)
    ops: list[HaloOp] = []
    if kind == "fg":
        for d in ("f", "g"):
            ops += [HaloOp("send", up, d, c, nzl) for c in CZ_UP]
        for d in ("f", "g"):
            ops += [HaloOp("send", down, d, c, 1) for c in CZ_DOWN]
        for d in ("f", "g"):
            ops += [HaloOp("recv", down, d, c, 0) for c in CZ_UP]
        for d in ("f", "g"):
            ops += [HaloOp("recv", up, d, c, nzl + 1) for c in CZ_DOWN]
    elif kind == "phi":
        ops = [HaloOp("send", up, kind, 0, nzl), HaloOp("send", down, kind, 0, 1),
               HaloOp("recv", down, kind, 0, 0), HaloOp("recv", up, kind, 0, nzl + 1)]
    else:
        ops = [HaloOp("send", up, kind, 0, nzl), HaloOp("send", down, kind, 0, 2),
               HaloOp("recv", down, kind, 0, 0), HaloOp("recv", up, kind, 0, nzl + 2)]
    return ops


def match_schedules(nranks: int, nzl: int, kind: str = "fg") -> list[tuple[HaloOp, int, HaloOp]]:
    """Pair every send with the receive it meets under per-peer FIFO matching.

    Returns [(send, receiver_rank, recv)]; raises if any pair disagrees on the
    payload (component / distribution) -- the property NCCL needs.
    """
    scheds = [halo_schedule(kind, r, nranks, nzl) for r in range(nranks)]
    pairs = []
    for r in range(nranks):
        sends = {}
        for op in scheds[r]:
            if op.op == "send":
                sends.setdefault(op.peer, []).append(op)
        for peer, lst in sends.items():
            recvs = [op for op in scheds[peer] if op.op == "recv" and op.peer == r]
            if len(recvs) != len(lst):
                raise ShapeError(f"rank {r} -> {peer}: {len(lst)} sends, {len(recvs)} recvs")
            for s, v in zip(lst, recvs):
                if (s.kind, s.comp) != (v.kind, v.comp):
                    raise ShapeError(f"mismatched halo pair {s} -> {v}")
                pairs.append((s, peer, v))
    return pairs


class VirtualSlabs:
    """P z-slabs of one lattice on one device, stepped through the C ABI."""

    def __init__(self, shape: LatticeShape, nslabs: int, params: nat.FluidParams,
                 vvl: int = 1, device: int = 0) -> None:
        if params.physics == 2:
            raise ConfigError("VirtualSlabs drives the C-ABI kernels (phi, mu, collide-stream); "
                              "the stress form (physics 2) runs through BinaryFluid only")
        self.shape, self.P, self.params, self.vvl = shape, nslabs, params, vvl
        nat.check(nat.lib.ltk_set_device(device))
        self.stream = nat.stream_create()
        z0, nzl = slab_bounds(shape.nz, 0, nslabs)
        if nzl < 2:
            raise ShapeError("z-slabs need >= 2 planes each (mu halos are 2 deep)")
        PL = shape.nx * shape.ny
        self.nzl, self.PL = nzl, PL
        cstride = -(-((nzl + 2) * PL) // 64) * 64
        self.slab = nat.Slab(shape.nx, shape.ny, nzl, cstride)
        self._ptrs = []
        self.bufs = []
        for _ in range(nslabs):
            b = {k: self._alloc(8 * Q * cstride) for k in ("fA", "gA", "fB", "gB")}
            b["phi"] = self._alloc(8 * (nzl + 2) * PL)
            b["mu"] = self._alloc(8 * (nzl + 4) * PL)
            self.bufs.append(b)
        self.face = self._alloc(8 * 10 * PL)
        self._stage, self._stage_bytes = 0, 0
        self.cur = "A"

    def _alloc(self, nbytes: int) -> int:
        p = nat.malloc(nbytes)
        self._ptrs.append(p)
        return p

    def close(self) -> None:
        nat.lib.ltk_stream_sync(self.stream)
        for p in self._ptrs:
            nat.free(p)
        self._ptrs = []
        nat.lib.ltk_stream_destroy(self.stream)

    def _staging(self, desc: FieldDescriptor) -> int:
        """One device staging buffer, reused by every load()/fields()."""
        if 2 * desc.nbytes > self._stage_bytes:
            if self._stage:
                nat.check(nat.lib.ltk_stream_sync(self.stream))
                self._ptrs.remove(self._stage)
                nat.free(self._stage)
            self._stage, self._stage_bytes = self._alloc(2 * desc.nbytes), 2 * desc.nbytes
        return self._stage

    def load(self, f: Field, g: Field) -> None:
        desc = f.descriptor
        if desc.nsites != self.shape.nsites:
            raise ShapeError("fields must cover the whole lattice")
        st = self._staging(desc)
        nb = desc.nbytes
        nat.check(nat.lib.ltk_h2d(st, f.data.ctypes.data, nb, self.stream))
        nat.check(nat.lib.ltk_h2d(st + nb, g.data.ctypes.data, nb, self.stream))
        for r, b in enumerate(self.bufs):
            z0, _ = slab_bounds(self.shape.nz, r, self.P)
            for src, dst in ((st, b["fA"]), (st + nb, b["gA"])):
                nat.check(nat.lib.ltk_fluid_scatter(ctypes.byref(self.slab), src,
                                                    desc.padded_sites, self.shape.nz, z0, Q,
                                                    dst, self.stream), "scatter")
        nat.check(nat.lib.ltk_stream_sync(self.stream))
        self.cur = "A"

    def fields(self) -> tuple[Field, Field]:
        desc = FieldDescriptor.create(Q, self.shape.nsites)
        st = self._staging(desc)
        nb = desc.nbytes
        for r, b in enumerate(self.bufs):
            z0, _ = slab_bounds(self.shape.nz, r, self.P)
            for src, dst in ((b["f" + self.cur], st), (b["g" + self.cur], st + nb)):
                nat.check(nat.lib.ltk_fluid_gather(ctypes.byref(self.slab), src,
                                                   desc.padded_sites, self.shape.nz, z0, Q,
                                                   dst, self.stream), "gather")
        f, g = field_create(desc), field_create(desc)
        nat.check(nat.lib.ltk_d2h(f.data.ctypes.data, st, nb, self.stream))
        nat.check(nat.lib.ltk_d2h(g.data.ctypes.data, st + nb, nb, self.stream))
        nat.check(nat.lib.ltk_stream_sync(self.stream))
        return f, g

    # -- halo exchange: the schedule of halo_schedule(), executed by copies ----

    def _exchange_fg(self, s: str) -> None:
        sl = ctypes.byref(self.slab)
        for r, b in enumerate(self.bufs):
            up, down = neighbours(r, self.P)
            for direction, peer in ((+1, up), (-1, down)):
                nat.check(nat.lib.ltk_fluid_pack_face(sl, b["f" + s], b["g" + s], self.face,
                                                      direction, self.stream))
                pb = self.bufs[peer]
                nat.check(nat.lib.ltk_fluid_unpack_face(sl, pb["f" + s], pb["g" + s], self.face,
                                                        direction, self.stream))

    def _exchange_plane(self, key: str) -> None:
        """phi: one plane per face (zs = z + 1); mu: two (zs = z + 2)."""
        h = 1 if key == "phi" else 2
        nb = 8 * self.PL
        for r, b in enumerate(self.bufs):
            up, down = neighbours(r, self.P)
            top, bot = b[key] + self.nzl * nb, b[key] + h * nb  # planes nzl-h.., 0..
            nat.check(nat.lib.ltk_d2d(self.bufs[up][key], top, h * nb, self.stream))
            nat.check(nat.lib.ltk_d2d(self.bufs[down][key] + (self.nzl + h) * nb, bot, h * nb,
                                      self.stream))

    def run(self, nsteps: int) -> None:
        sl = ctypes.byref(self.slab)
        prm = ctypes.byref(self.params)
        for _ in range(nsteps):
            s, o = self.cur, ("B" if self.cur == "A" else "A")
            self._exchange_fg(s)
            for b in self.bufs:
                nat.check(nat.lib.ltk_fluid_phi(sl, b["g" + s], b["phi"], 0, self.nzl,
                                                self.stream), "phi")
            self._exchange_plane("phi")
            if self.params.physics == 1:
                for b in self.bufs:
                    nat.check(nat.lib.ltk_fluid_mu(sl, b["phi"], b["mu"], prm, 0, self.nzl,
                                                   self.stream), "mu")
                self._exchange_plane("mu")
            for b in self.bufs:
                nat.check(nat.lib.ltk_fluid_collide_stream(
                    sl, b["f" + s], b["g" + s], b["phi"], b["mu"], b["f" + o], b["g" + o], prm,
                    0, self.nzl, self.vvl, self.stream), "collide_stream")
            self.cur = o
        site = ctypes.c_int64(-1)
        rc = nat.lib.ltk_sync(self.stream, ctypes.byref(site))
        if rc == nat.LTK_ERR_SINGULAR:
            raise SingularStateError(f"rho <= 0 (slab-local site {site.value})")
        nat.check(rc)
