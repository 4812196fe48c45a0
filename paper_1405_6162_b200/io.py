"""Distributed field dump / load in the reference's on-disk format.

Format (reference pkg/src/latkit/lattice.py:172-198): little-endian
header (ncomp, nx, ny, nz) as four uint64, then the real-site doubles of each
component in host site order (x*ny + y)*nz + z.  A z-slab of planes
[z0, z0+nzl) is a strided sub-block of that layout, so every rank writes its
own block straight into the shared file through a memory map: no gather to
rank 0, and the file is byte-identical to `field_dump` of the whole field.
"""

from __future__ import annotations

import os
import struct
from typing import Callable

import numpy as np

from .errors import ShapeError
from .lattice import Field, FieldDescriptor, LatticeShape, field_create

_HEADER = struct.Struct("<4Q")


def create_field_file(path: str, ncomp: int, shape: LatticeShape) -> None:
    """Write the header and size the file (one rank)."""
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(ncomp, shape.nx, shape.ny, shape.nz))
        fh.truncate(_HEADER.size + 8 * ncomp * shape.nsites)


def read_header(path: str) -> tuple[int, LatticeShape]:
    with open(path, "rb") as fh:
        raw = fh.read(_HEADER.size)
    if len(raw) != _HEADER.size:
        raise ShapeError("truncated field header")
    ncomp, nx, ny, nz = _HEADER.unpack(raw)
    need = _HEADER.size + 8 * ncomp * nx * ny * nz
    if os.path.getsize(path) < need:
        raise ShapeError("truncated field body")
    return ncomp, LatticeShape(nx, ny, nz)


def _map(path: str, ncomp: int, shape: LatticeShape, mode: str) -> np.memmap:
    return np.memmap(path, dtype="<f8", mode=mode, offset=_HEADER.size,
                     shape=(ncomp, shape.nx, shape.ny, shape.nz))


def write_slab(path: str, slab: Field, shape: LatticeShape, z0: int) -> None:
    """Write a slab field (nx*ny*nzl sub-lattice, host order) into planes [z0, z0+nzl)."""
    ncomp, fshape = read_header(path)
    if fshape != shape or slab.descriptor.ncomp != ncomp:
        raise ShapeError(f"file holds {ncomp}x{fshape}, slab is {slab.descriptor.ncomp} "
                         f"components of {shape}")
    nzl = slab.descriptor.nsites // (shape.nx * shape.ny)
    if nzl * shape.nx * shape.ny != slab.descriptor.nsites or z0 + nzl > shape.nz:
        raise ShapeError("slab does not tile the lattice")
    mm = _map(path, ncomp, shape, "r+")
    body = slab.components()[:, :slab.descriptor.nsites]
    mm[:, :, :, z0:z0 + nzl] = body.reshape(ncomp, shape.nx, shape.ny, nzl)
    mm.flush()
    del mm


def read_slab(path: str, z0: int, nzl: int) -> tuple[Field, LatticeShape]:
    """Read planes [z0, z0+nzl) as an nx*ny*nzl host-order field."""
    ncomp, shape = read_header(path)
    if z0 < 0 or z0 + nzl > shape.nz:
        raise ShapeError("slab outside the lattice")
    mm = _map(path, ncomp, shape, "r")
    n = shape.nx * shape.ny * nzl
    out = field_create(FieldDescriptor.create(ncomp, n))
    out.components()[:, :n] = np.asarray(mm[:, :, :, z0:z0 + nzl]).reshape(ncomp, n)
    del mm
    return out, shape


def dump_state(sim, prefix: str, barrier: Callable[[], None] | None = None) -> tuple[str, str]:
    """Collective dump of a BinaryFluid's (f, g) to <prefix>.f / <prefix>.g."""
    barrier = barrier or (lambda: None)
    f, g = sim.fields(slab_only=True)
    paths = (prefix + ".f", prefix + ".g")
    if sim.rank == 0:
        for p in paths:
            create_field_file(p, 19, sim.shape)
    barrier()
    write_slab(paths[0], f, sim.shape, sim.z0)
    write_slab(paths[1], g, sim.shape, sim.z0)
    barrier()
    return paths


def load_state(sim, prefix: str) -> None:
    """Collective load of <prefix>.f / <prefix>.g into a BinaryFluid (each rank its slab)."""
    f, shape = read_slab(prefix + ".f", sim.z0, sim.nzl)
    g, _ = read_slab(prefix + ".g", sim.z0, sim.nzl)
    if shape != sim.shape:
        raise ShapeError(f"file lattice {shape} != engine lattice {sim.shape}")
    sim.load(f, g)
