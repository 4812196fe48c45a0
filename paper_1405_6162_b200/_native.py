"""ctypes binding of libltk.so (include/ltk.h).

The product path has no CPU fallback: if the shared library is missing this
module raises at import time, and every compute call goes through the CUDA
kernels in csrc/.  ctypes releases the GIL during each call.
"""

from __future__ import annotations

import ctypes
import os

from .errors import (AllocationError, BoundsError, ConfigError, DeviceError, LatkitError,
                     LifecycleError, PlanError, ShapeError, SingularStateError)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_native", "libltk.so")
Q = 19

LTK_OK = 0
IPC_BLOB_BYTES = 1024
ABI_VERSION = 2
LTK_ERR_SINGULAR = 11
MODE_EXACT = 0
MODE_FAST = 1
MU_AUTO, MU_PLAIN = 0, 1
LAYOUT_SOA, LAYOUT_ROW = 0, 1

_ERRORS = {1: ConfigError, 2: BoundsError, 3: ShapeError, 4: AllocationError,
           5: LifecycleError, 6: PlanError, 7: DeviceError, 11: SingularStateError}

_i32, _i64, _dbl, _vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
_pp = ctypes.POINTER(ctypes.c_void_p)


class CollisionParams(ctypes.Structure):
    """ltk_collision_params."""

    _fields_ = [("wv", _dbl * Q), ("cs2", _dbl), ("tau_f", _dbl), ("tau_g", _dbl),
                ("mode", _i32), ("reserved", _i32)]


class FluidParams(ctypes.Structure):
    """ltk_fluid_params."""

    _fields_ = [("wv", _dbl * Q), ("lam", _dbl * Q), ("cs2", _dbl), ("tau_f", _dbl),
                ("tau_g", _dbl), ("A", _dbl), ("B", _dbl), ("kappa", _dbl), ("gamma", _dbl),
                ("physics", _i32), ("mode", _i32)]


class Slab(ctypes.Structure):
    """ltk_slab."""

    _fields_ = [("nx", _i64), ("ny", _i64), ("nzl", _i64), ("cstride", _i64)]


# name -> (restype, argtypes); every symbol of include/ltk.h
SIGNATURES = {
    "ltk_abi_version": (ctypes.c_int, []),
    "ltk_last_error": (ctypes.c_char_p, []),
    "ltk_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "ltk_set_device": (ctypes.c_int, [ctypes.c_int]),
    "ltk_get_device": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "ltk_device_info": (ctypes.c_int, [ctypes.c_int, ctypes.c_char_p,
                                       ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_i64),
                                       ctypes.POINTER(ctypes.c_int),
                                       ctypes.POINTER(ctypes.c_int)]),
    "ltk_malloc": (ctypes.c_int, [_pp, ctypes.c_size_t]),
    "ltk_free": (ctypes.c_int, [_vp]),
    "ltk_mem_info": (ctypes.c_int, [ctypes.POINTER(ctypes.c_size_t),
                                    ctypes.POINTER(ctypes.c_size_t)]),
    "ltk_memset0": (ctypes.c_int, [_vp, ctypes.c_size_t, _vp]),
    "ltk_h2d": (ctypes.c_int, [_vp, _vp, ctypes.c_size_t, _vp]),
    "ltk_d2h": (ctypes.c_int, [_vp, _vp, ctypes.c_size_t, _vp]),
    "ltk_d2d": (ctypes.c_int, [_vp, _vp, ctypes.c_size_t, _vp]),
    "ltk_host_register": (ctypes.c_int, [_vp, ctypes.c_size_t]),
    "ltk_host_unregister": (ctypes.c_int, [_vp]),
    "ltk_host_alloc": (ctypes.c_int, [_pp, ctypes.c_size_t]),
    "ltk_host_free": (ctypes.c_int, [_vp]),
    "ltk_stream_create": (ctypes.c_int, [_pp]),
    "ltk_stream_destroy": (ctypes.c_int, [_vp]),
    "ltk_stream_sync": (ctypes.c_int, [_vp]),
    "ltk_event_create": (ctypes.c_int, [_pp, ctypes.c_int]),
    "ltk_event_destroy": (ctypes.c_int, [_vp]),
    "ltk_event_record": (ctypes.c_int, [_vp, _vp]),
    "ltk_event_query": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int)]),
    "ltk_event_sync": (ctypes.c_int, [_vp]),
    "ltk_event_elapsed": (ctypes.c_int, [_vp, _vp, ctypes.POINTER(ctypes.c_float)]),
    "ltk_stream_wait_event": (ctypes.c_int, [_vp, _vp]),
    "ltk_sync": (ctypes.c_int, [_vp, ctypes.POINTER(_i64)]),
    "ltk_launch_count": (_i64, []),
    "ltk_scale": (ctypes.c_int, [_i64, _i64, _i32, _i32, _vp, _i64, _dbl, _vp]),
    "ltk_collide": (ctypes.c_int, [_i64, _i64, _i32, _i32, _vp, _vp, _i64, _i64,
                                   ctypes.POINTER(CollisionParams), _vp]),
    "ltk_pack_sites": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i32, _i64, _vp]),
    "ltk_unpack_sites": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i32, _i64, _vp]),
    "ltk_fluid_phi": (ctypes.c_int, [ctypes.POINTER(Slab), _vp, _vp, _i64, _i64, _vp]),
    "ltk_fluid_mu": (ctypes.c_int, [ctypes.POINTER(Slab), _vp, _vp, ctypes.POINTER(FluidParams),
                                    _i64, _i64, _vp]),
    "ltk_fluid_collide_stream": (ctypes.c_int, [ctypes.POINTER(Slab), _vp, _vp, _vp, _vp, _vp,
                                                _vp, ctypes.POINTER(FluidParams), _i64, _i64,
                                                _i32, _vp]),
    "ltk_fluid_wrap_halos": (ctypes.c_int, [ctypes.POINTER(Slab), _vp, _vp, _vp, _vp, _i32,
                                            _vp]),
    "ltk_fluid_pack_face": (ctypes.c_int, [ctypes.POINTER(Slab), _vp, _vp, _vp, _i32, _vp]),
    "ltk_fluid_unpack_face": (ctypes.c_int, [ctypes.POINTER(Slab), _vp, _vp, _vp, _i32, _vp]),
    "ltk_fluid_scatter": (ctypes.c_int, [ctypes.POINTER(Slab), _vp, _i64, _i64, _i64, _i32, _vp,
                                         _vp]),
    "ltk_fluid_gather": (ctypes.c_int, [ctypes.POINTER(Slab), _vp, _i64, _i64, _i64, _i32, _vp,
                                        _vp]),
    "ltk_fluid_create": (ctypes.c_int, [_i64, _i64, _i64, _i32, _i32,
                                        ctypes.POINTER(FluidParams), _i32, _pp]),
    "ltk_fluid_destroy": (ctypes.c_int, [_vp]),
    "ltk_fluid_slab": (ctypes.c_int, [_vp, ctypes.POINTER(Slab), ctypes.POINTER(_i64)]),
    "ltk_fluid_buffers": (ctypes.c_int, [_vp, _pp, _pp, _pp, _pp]),
    "ltk_fluid_set_params": (ctypes.c_int, [_vp, ctypes.POINTER(FluidParams)]),
    "ltk_fluid_stream": (ctypes.c_int, [_vp, _pp]),
    "ltk_fluid_load": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "ltk_fluid_store": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "ltk_fluid_run": (ctypes.c_int, [_vp, _i64, _vp]),
    "ltk_fluid_totals": (ctypes.c_int, [_vp, ctypes.POINTER(_dbl)]),
    "ltk_fluid_use_graph": (ctypes.c_int, [_vp, _i32]),
    "ltk_fluid_sync": (ctypes.c_int, [_vp, ctypes.POINTER(_i64)]),
    "ltk_div_selftest": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp, _vp]),
    "ltk_fluid_mu_variant": (ctypes.c_int, [_i32, ctypes.POINTER(_i32)]),
    "ltk_fluid_set_layout": (ctypes.c_int, [_vp, _i32, ctypes.POINTER(_i32)]),
    "ltk_fluid_profile": (ctypes.c_int, [_vp, _i32, ctypes.POINTER(ctypes.c_float)]),
    "ltk_fluid_ipc_blob": (ctypes.c_int, [_vp, ctypes.c_char_p]),
    "ltk_fluid_attach_peers": (ctypes.c_int, [_vp, ctypes.c_char_p, ctypes.c_char_p]),
    "ltk_fluid_attach_peer_engines": (ctypes.c_int, [_vp, _vp, _vp]),
    "ltk_fluid_peer_timeout": (ctypes.c_int, [_vp, ctypes.POINTER(_i32)]),
    "ltk_fluid_inject_peer_timeout": (ctypes.c_int, [_vp]),
    "ltk_nccl_available": (ctypes.c_int, []),
    "ltk_nccl_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
    "ltk_fluid_attach_nccl": (ctypes.c_int, [_vp, ctypes.c_char_p]),
}


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libltk.so not found at {LIB_PATH}: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    missing = []
    for name, (res, args) in SIGNATURES.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            missing.append(name)
            continue
        fn.restype = res
        fn.argtypes = args
    if missing:
        raise ImportError(f"libltk.so lacks symbols {missing}: rebuild it")
    if lib.ltk_abi_version() != ABI_VERSION:
        raise ImportError(f"libltk.so ABI {lib.ltk_abi_version()} != {ABI_VERSION}: rebuild it")
    return lib


lib = _load()


def last_error() -> str:
    msg = lib.ltk_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(rc: int, what: str = "") -> None:
    """Raise the framework exception mapped from an ltk_status."""
    if rc != LTK_OK:
        exc = _ERRORS.get(rc, LatkitError)
        detail = last_error()
        raise exc(f"{what}: {detail}" if what else detail)


def malloc(nbytes: int) -> int:
    p = ctypes.c_void_p()
    check(lib.ltk_malloc(ctypes.byref(p), nbytes), "ltk_malloc")
    return int(p.value)


def free(ptr: int) -> None:
    check(lib.ltk_free(ptr), "ltk_free")


def stream_create() -> int:
    s = ctypes.c_void_p()
    check(lib.ltk_stream_create(ctypes.byref(s)), "ltk_stream_create")
    return int(s.value)


def event_create(timing: bool = False) -> int:
    e = ctypes.c_void_p()
    check(lib.ltk_event_create(ctypes.byref(e), 1 if timing else 0), "ltk_event_create")
    return int(e.value)


def event_done(event: int) -> bool:
    d = ctypes.c_int(0)
    check(lib.ltk_event_query(event, ctypes.byref(d)), "ltk_event_query")
    return bool(d.value)


def elapsed_ms(start: int, stop: int) -> float:
    ms = ctypes.c_float()
    check(lib.ltk_event_elapsed(start, stop, ctypes.byref(ms)), "ltk_event_elapsed")
    return float(ms.value)


def device_count() -> int:
    n = ctypes.c_int(0)
    rc = lib.ltk_device_count(ctypes.byref(n))
    return int(n.value) if rc == LTK_OK else 0


def launch_count() -> int:
    return int(lib.ltk_launch_count())
