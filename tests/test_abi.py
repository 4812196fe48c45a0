"""The C-ABI boundary on CPU: libltk.so loads, exports exactly what
include/ltk.h declares, and the ctypes layer binds all of it (no GPU calls)."""

import os
import re
import subprocess

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "ltk.h")
LIB = os.path.join(ROOT, "paper_1405_6162_b200", "_native", "libltk.so")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(ltk_[a-z0-9_]+)\s*\(", text))


def test_header_declares_the_api():
    names = declared()
    for must in ("ltk_collide", "ltk_scale", "ltk_malloc", "ltk_h2d", "ltk_d2h", "ltk_sync",
                 "ltk_fluid_collide_stream", "ltk_fluid_phi", "ltk_fluid_mu", "ltk_fluid_run",
                 "ltk_pack_sites", "ltk_fluid_attach_nccl"):
        assert must in names


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (ltk_[a-z0-9_]+)$", out, flags=re.M))
    assert declared() <= exported, declared() - exported
    assert exported <= declared(), exported - declared()


def test_ctypes_binding_covers_header():
    from paper_1405_6162_b200 import _native as nat

    assert set(nat.SIGNATURES) == declared()
    assert nat.lib.ltk_abi_version() == 1


def test_struct_layouts_match_header():
    from paper_1405_6162_b200 import _native as nat
    import ctypes

    assert ctypes.sizeof(nat.CollisionParams) == 19 * 8 + 3 * 8 + 8
    assert ctypes.sizeof(nat.FluidParams) == 2 * 19 * 8 + 7 * 8 + 8
    assert ctypes.sizeof(nat.Slab) == 32


def test_sm100a_code_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_no_gpu_means_loud_failure():
    import pytest

    import paper_1405_6162_b200 as lk
    from conftest import gpu_available

    if gpu_available():
        pytest.skip("GPU present")
    with pytest.raises(lk.ConfigError):
        lk.TargetDevice()
    with pytest.raises(lk.ConfigError):
        lk.BinaryFluid(lk.LatticeShape(4, 4, 4))
