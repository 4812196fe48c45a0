"""Full D3Q19 binary-fluid timestep on B200 (north-star extension).

The reference stops at the collision (reference pkg/README.md:34-35); this
module adds the timestep of SURVEY.md Appendix C, specified in DESIGN.md §2:

    stream (pull) -> phi = sum g -> mu = A phi + B phi^3 - kappa lap(phi)
    -> Guo-forced collision of f with the potential force -phi grad(mu)
       (each component filtered [1/4 1/2 1/4] along its own axis, which keeps
       flat interfaces at rest: DESIGN.md §2), g relaxed to an equilibrium
       carrying the chemical potential.

`BinaryFluid` owns one z-slab (the whole lattice on one GPU) in the C++
engine of csrc/fluid.cu and runs whole timesteps without Python in the loop.
With `physics="passive"` the collision is exactly the reference collision
(kernels.py:89-125) applied after streaming.

Host fields use the reference layout (Field, site (x*ny + y)*nz + z); the
device keeps a z-slowest slab with halo planes and converts
with on-device transposes.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import ConfigError, ShapeError, SingularStateError
from .lattice import Field, FieldDescriptor, LatticeShape, field_create
from .model import D3Q19Model, Q

MODE_EXACT = nat.MODE_EXACT
MODE_FAST = nat.MODE_FAST
MU_AUTO, MU_PLAIN = nat.MU_AUTO, nat.MU_PLAIN
LAYOUT_SOA, LAYOUT_ROW = nat.LAYOUT_SOA, nat.LAYOUT_ROW
#: passive: the reference collision after streaming; binary: free-energy binary
#: fluid with the filtered potential force -phi grad(mu) (flat interfaces relax
#: to rest); binary-stress: the same fluid with the momentum-conserving
#: F = -div P of the chemical pressure tensor (Ludwig's divergence form; its
#: discrete force is not zero at equilibrium: spurious currents ~1e-4)
PHYSICS = {"passive": 0, "binary": 1, "binary-stress": 2}


@dataclass(frozen=True)
class FreeEnergy:
    """Symmetric binary free energy f = A/2 phi^2 + B/4 phi^4 + kappa/2 |grad phi|^2.

    Defaults give phi* = +-1 and interface width xi = sqrt(-2 kappa / A) ~ 1.13
    (SURVEY.md Appendix C).  gamma is the mobility parameter of g_eq.
    """

    A: float = -0.0625
    B: float = 0.0625
    kappa: float = 0.04
    gamma: float = 1.0


def lam_weights(model: D3Q19Model) -> np.ndarray:
    """lam_i = w_i/cs2 (i > 0), lam_0 = -(1 - w_0)/cs2: sum lam = 0,
    sum lam c = 0, sum lam c c = I, so sum g_eq c c = gamma mu I + phi u u."""
    lam = np.array([w / model.cs2 for w in model.wv])
    lam[0] = -(1.0 - model.wv[0]) / model.cs2
    return lam


def fluid_params(model: D3Q19Model | None = None, free_energy: FreeEnergy | None = None,
                 physics: str = "binary", mode: int = MODE_EXACT) -> nat.FluidParams:
    model = model or D3Q19Model()
    fe = free_energy or FreeEnergy()
    if physics not in PHYSICS:
        raise ConfigError(f"physics must be one of {tuple(PHYSICS)}, got {physics!r}")
    if mode not in (MODE_EXACT, MODE_FAST):
        raise ConfigError(f"mode must be MODE_EXACT or MODE_FAST, got {mode}")
    p = nat.FluidParams()
    lam = lam_weights(model)
    for i in range(Q):
        p.wv[i] = float(model.wv[i])
        p.lam[i] = float(lam[i])
    p.cs2, p.tau_f, p.tau_g = float(model.cs2), float(model.tau_f), float(model.tau_g)
    p.A, p.B, p.kappa, p.gamma = float(fe.A), float(fe.B), float(fe.kappa), float(fe.gamma)
    p.physics, p.mode = PHYSICS[physics], int(mode)
    return p


class _Scratch:
    """Device staging buffer in reference site order (load/store transposes)."""

    def __init__(self) -> None:
        self.ptr, self.nbytes = 0, 0

    def get(self, nbytes: int) -> int:
        if nbytes > self.nbytes:
            self.release()
            self.ptr, self.nbytes = nat.malloc(nbytes), nbytes
        return self.ptr

    def release(self) -> None:
        if self.ptr:
            nat.free(self.ptr)
            self.ptr, self.nbytes = 0, 0


class BinaryFluid:
    """One z-slab of a periodic nx*ny*nz lattice, resident on one B200.

    nranks == 1: the whole lattice, periodic z wrap inside the kernels.
    nranks > 1: planes [rank*nz/nranks, (rank+1)*nz/nranks); call
    `attach_nccl(unique_id)` (bytes from `nccl_unique_id()` on rank 0,
    broadcast by the caller) before stepping.
    """

    def __init__(self, shape: LatticeShape, model: D3Q19Model | None = None,
                 free_energy: FreeEnergy | None = None, physics: str = "binary",
                 mode: int = MODE_EXACT, vvl: int = 1, rank: int = 0, nranks: int = 1,
                 device: int = 0, use_graph: bool = True) -> None:
        self.shape = shape
        self.model = model or D3Q19Model()
        self.free_energy = free_energy or FreeEnergy()
        self.physics, self.mode, self.vvl = physics, mode, vvl
        self.rank, self.nranks, self.device = rank, nranks, device
        if nat.device_count() <= device:
            raise ConfigError(f"no CUDA device {device}: BinaryFluid runs only on the GPU")
        nat.check(nat.lib.ltk_set_device(device), "ltk_set_device")
        self._params = fluid_params(self.model, self.free_energy, physics, mode)
        h = ctypes.c_void_p()
        nat.check(nat.lib.ltk_fluid_create(shape.nx, shape.ny, shape.nz, rank, nranks,
                                           ctypes.byref(self._params), vvl, ctypes.byref(h)),
                  "ltk_fluid_create")
        self._h = h.value
        self.slab = nat.Slab()
        z0 = ctypes.c_int64()
        nat.lib.ltk_fluid_slab(self._h, ctypes.byref(self.slab), ctypes.byref(z0))
        self.z0 = int(z0.value)
        self.nzl = int(self.slab.nzl)
        self._scratch = _Scratch()
        st = ctypes.c_void_p()
        nat.check(nat.lib.ltk_fluid_stream(self._h, ctypes.byref(st)), "ltk_fluid_stream")
        self.stream = st.value
        self.steps_done = 0
        self.set_graph(use_graph and nranks == 1)

    # -- lifecycle -----------------------------------------------------------

    def close(self) -> None:
        if getattr(self, "_h", None):
            nat.lib.ltk_set_device(self.device)
            nat.lib.ltk_fluid_destroy(self._h)
            self._h = None
            self._scratch.release()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> int:
        return self._h

    def set_graph(self, enable: bool) -> None:
        nat.check(nat.lib.ltk_fluid_use_graph(self._h, 1 if enable else 0), "use_graph")

    def set_layout(self, layout: int | None = None) -> int:
        """f/g storage layout of this slab: LAYOUT_ROW (row-blocked: the 19
        components of an x-row adjacent; default for even nx, measured faster)
        or LAYOUT_SOA (component-major planes).  Every transport takes either.
        Bitwise identical results; set before load() and before attaching a
        transport.  Returns the previous layout (None only queries)."""
        prev = ctypes.c_int32()
        nat.check(nat.lib.ltk_fluid_set_layout(self._h, -1 if layout is None else int(layout),
                                               ctypes.byref(prev)), "set_layout")
        return prev.value

    def ipc_blob(self) -> bytes:
        """CUDA IPC handles of this slab's buffers (exchange them, then attach_peers)."""
        buf = ctypes.create_string_buffer(nat.IPC_BLOB_BYTES)
        nat.check(nat.lib.ltk_fluid_ipc_blob(self._h, buf), "ltk_fluid_ipc_blob")
        return buf.raw

    def attach_peers(self, up_blob: bytes, down_blob: bytes) -> None:
        """Peer transport: halo images are stored by the kernels straight into
        the slabs above/below over NVLink.  All ranks must attach before any
        rank loads (put a barrier between the two)."""
        nat.check(nat.lib.ltk_fluid_attach_peers(self._h, up_blob, down_blob), "attach_peers")

    def attach_peer_engines(self, up: "BinaryFluid", down: "BinaryFluid") -> None:
        """Peer transport between engines of this process (e.g. one thread
        driving several GPUs, or several slabs of one GPU)."""
        nat.check(nat.lib.ltk_fluid_attach_peer_engines(self._h, up.handle, down.handle),
                  "attach_peer_engines")

    def peer_timed_out(self) -> bool:
        v = ctypes.c_int32(0)
        nat.check(nat.lib.ltk_fluid_peer_timeout(self._h, ctypes.byref(v)), "peer_timeout")
        return bool(v.value)

    def inject_peer_timeout(self) -> None:
        """Test hook: the next progress waits fail at once, as if a neighbour
        had stalled; sync() then raises DeviceError."""
        nat.check(nat.lib.ltk_fluid_inject_peer_timeout(self._h), "inject_peer_timeout")

    def attach_nccl(self, unique_id: bytes) -> None:
        if len(unique_id) != 128:
            raise ConfigError("NCCL unique id must be 128 bytes")
        nat.check(nat.lib.ltk_fluid_attach_nccl(self._h, unique_id), "attach_nccl")

    # -- state transfer --------------------------------------------------------

    def _src_geometry(self, nsites_src: int) -> tuple[int, int]:
        """(nz_src, z_src0) for a host array of nsites_src sites."""
        s = self.shape
        if nsites_src == s.nsites:
            return s.nz, self.z0
        if nsites_src == s.nx * s.ny * self.nzl:
            return self.nzl, 0
        raise ShapeError(f"field has {nsites_src} sites; expected the lattice "
                         f"({s.nsites}) or this slab ({s.nx * s.ny * self.nzl})")

    def load(self, f: Field, g: Field) -> None:
        """Upload reference-ordered host fields (whole lattice, or this slab only)."""
        if f.descriptor != g.descriptor or f.descriptor.ncomp != Q:
            raise ShapeError("f and g must be 19-component fields with one descriptor")
        nz_src, z_src0 = self._src_geometry(f.descriptor.nsites)
        nb = f.descriptor.nbytes
        base = self._scratch.get(2 * nb)
        nat.check(nat.lib.ltk_set_device(self.device))
        nat.check(nat.lib.ltk_h2d(base, f.data.ctypes.data, nb, self.stream), "H2D f")
        nat.check(nat.lib.ltk_h2d(base + nb, g.data.ctypes.data, nb, self.stream), "H2D g")
        nat.check(nat.lib.ltk_fluid_load(self._h, base, base + nb, f.descriptor.padded_sites,
                                         nz_src, z_src0, self.stream), "ltk_fluid_load")
        self.sync()
        self.steps_done = 0

    def load_device(self, f_ptr: int, g_ptr: int, padded: int, nz_src: int, z_src0: int,
                    stream: int | None = None) -> None:
        """Load from reference-ordered arrays already in device memory (no sync)."""
        nat.check(nat.lib.ltk_fluid_load(self._h, f_ptr, g_ptr, padded, nz_src, z_src0, stream),
                  "ltk_fluid_load")

    def store_device(self, f_ptr: int, g_ptr: int, padded: int, nz_src: int, z_src0: int,
                     stream: int | None = None) -> None:
        nat.check(nat.lib.ltk_fluid_store(self._h, f_ptr, g_ptr, padded, nz_src, z_src0, stream),
                  "ltk_fluid_store")

    def fields(self, slab_only: bool | None = None) -> tuple[Field, Field]:
        """Download the current state in reference order.

        Whole lattice when nranks == 1; otherwise this slab's planes as an
        nx*ny*nzl sub-lattice (slab_only defaults to nranks > 1)."""
        if slab_only is None:
            slab_only = self.nranks > 1
        s = self.shape
        if slab_only:
            nsites, nz_src, z_src0 = s.nx * s.ny * self.nzl, self.nzl, 0
        else:
            if self.nranks > 1:
                raise ShapeError("a single slab cannot produce the whole lattice")
            nsites, nz_src, z_src0 = s.nsites, s.nz, 0
        desc = FieldDescriptor.create(Q, nsites)
        f, g = field_create(desc), field_create(desc)
        nb = desc.nbytes
        base = self._scratch.get(2 * nb)
        nat.check(nat.lib.ltk_set_device(self.device))
        nat.check(nat.lib.ltk_memset0(base, 2 * nb, self.stream))
        nat.check(nat.lib.ltk_fluid_store(self._h, base, base + nb, desc.padded_sites, nz_src,
                                          z_src0, self.stream), "ltk_fluid_store")
        nat.check(nat.lib.ltk_d2h(f.data.ctypes.data, base, nb, self.stream), "D2H f")
        nat.check(nat.lib.ltk_d2h(g.data.ctypes.data, base + nb, nb, self.stream), "D2H g")
        self.sync()
        return f, g

    def order_parameter(self) -> tuple[np.ndarray, np.ndarray]:
        """(phi, mu) of the last step over the owned planes, shape (nzl, ny, nx)."""
        s = self.shape
        PL = s.nx * s.ny
        ptrs = [ctypes.c_void_p() for _ in range(4)]
        nat.lib.ltk_fluid_buffers(self._h, *[ctypes.byref(p) for p in ptrs])
        out = []
        for p, halo in ((ptrs[2], 1), (ptrs[3], 2)):  # phi: 1 halo plane per face, mu: 2
            a = np.empty((self.nzl + 2 * halo) * PL)
            nat.check(nat.lib.ltk_d2h(a.ctypes.data, p.value, a.nbytes, self.stream), "D2H")
            out.append(a[halo * PL:(self.nzl + halo) * PL].reshape(self.nzl, s.ny, s.nx))
        self.sync()
        return tuple(out)

    def totals(self, allreduce=None) -> np.ndarray:
        """[sum rho, sum j_x, sum j_y, sum j_z, sum phi] of the current state on
        the device (no state copy).  `allreduce(np.ndarray) -> np.ndarray`
        sums the slabs of a multi-GPU run (e.g. torch.distributed)."""
        out = (ctypes.c_double * 5)()
        nat.check(nat.lib.ltk_fluid_totals(self._h, out), "ltk_fluid_totals")
        tot = np.array(out[:])
        return allreduce(tot) if allreduce is not None else tot

    def set_model(self, model: D3Q19Model | None = None, free_energy: FreeEnergy | None = None,
                  physics: str | None = None, mode: int | None = None) -> None:
        """Change relaxation times, free energy, force form or arithmetic mode
        between steps (the state stays; later steps use the new parameters)."""
        self.model = model or self.model
        self.free_energy = free_energy or self.free_energy
        self.physics = physics or self.physics
        self.mode = self.mode if mode is None else mode
        self._params = fluid_params(self.model, self.free_energy, self.physics, self.mode)
        nat.check(nat.lib.ltk_fluid_set_params(self._h, ctypes.byref(self._params)),
                  "ltk_fluid_set_params")

    # -- stepping ------------------------------------------------------------

    def run(self, nsteps: int, stream: int | None = None) -> None:
        """Enqueue `nsteps` timesteps (asynchronous; errors surface at sync())."""
        nat.check(nat.lib.ltk_set_device(self.device))
        nat.check(nat.lib.ltk_fluid_run(self._h, int(nsteps), stream), "ltk_fluid_run")
        self.steps_done += int(nsteps)

    def sync(self) -> None:
        """Wait for the engine's streams and check its own error words:
        SingularStateError on rho <= 0 (lowest site, host order), DeviceError
        when a peer progress wait timed out (a neighbour slab stalled; the
        engine then refuses further steps)."""
        site = ctypes.c_int64(-1)
        rc = nat.lib.ltk_fluid_sync(self._h, ctypes.byref(site))
        if rc == nat.LTK_ERR_SINGULAR:
            raise SingularStateError(f"rho <= 0 at lattice site {site.value}")
        nat.check(rc, "sync")

    def profile(self, enable: bool) -> list[float]:
        """Toggle per-kernel event timing; returns accumulated ms of the last
        window: [phi, mu (+halo), collide_stream (+halo), whole step]."""
        arr = (ctypes.c_float * 4)()
        nat.check(nat.lib.ltk_fluid_profile(self._h, 1 if enable else 0, arr), "profile")
        return [float(v) for v in arr]


def mu_variant(variant: int | None = None) -> int:
    """Chemical-potential stencil kernel of the process: MU_AUTO (the
    shared-memory tile kernel k_mu_tile where the shape allows it, else the
    plain one) or MU_PLAIN.  Bitwise identical.
    Returns the previous value; None only queries."""
    prev = ctypes.c_int32(0)
    nat.check(nat.lib.ltk_fluid_mu_variant(-1 if variant is None else int(variant),
                                           ctypes.byref(prev)), "mu_variant")
    return int(prev.value)


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0); broadcast it with torch.distributed."""
    buf = ctypes.create_string_buffer(128)
    nat.check(nat.lib.ltk_nccl_unique_id(buf), "ltk_nccl_unique_id")
    return buf.raw


def nccl_available() -> bool:
    return bool(nat.lib.ltk_nccl_available())
