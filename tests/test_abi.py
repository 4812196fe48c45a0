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
    assert nat.lib.ltk_abi_version() == nat.ABI_VERSION == 2


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


def test_plain_c_host_compiles_and_links(tmp_path):
    # include/ltk.h is a C header: a C99 host (the paper's targetDP setting,
    # INTEGRATION.md §2) compiles against it and links libltk.so
    src = tmp_path / "host.c"
    src.write_text(r"""
#include <stdio.h>
#include "ltk.h"
int main(void) {
    ltk_collision_params p = {{0}, 1.0 / 3.0, 1.0, 1.0, LTK_MODE_EXACT, 0};
    ltk_fluid_params q;
    int64_t site = -1;
    int n = 0;
    (void)p; (void)q; (void)site;
    if (ltk_abi_version() != LTK_ABI_VERSION) return 1;
    if (ltk_device_count(&n) != LTK_OK && n != 0) return 2;
    printf("abi %d devices %d\n", ltk_abi_version(), n);
    return 0;
}
""")
    exe = tmp_path / "host"
    lib_dir = os.path.dirname(LIB)
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    str(src), "-L", lib_dir, "-lltk", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)],
                   check=True, capture_output=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert out.stdout.startswith("abi 2")


def test_nccl_shim_covers_the_engines_nccl_symbols(tmp_path):
    # the stand-in libnccl.so.2 of tests/nccl_shim (GPU test of the NCCL slab path
    # with P >= 2 ranks on one device) exports every symbol fluid.cu dlsym's
    src = open(os.path.join(ROOT, "paper_1405_6162_b200", "csrc", "fluid.cu")).read()
    wanted = set(re.findall(r'dlsym\(n\.h, "(nccl\w+)"\)', src))
    assert len(wanted) == 8
    out = tmp_path / "libnccl.so.2"
    subprocess.run(["g++", "-O2", "-fPIC", "-shared", "-Wl,-soname,libnccl.so.2",
                    "-I/usr/local/cuda/include", "-o", str(out),
                    os.path.join(ROOT, "tests", "nccl_shim", "nccl_shim.cpp"),
                    "-L/usr/local/cuda/lib64", "-lcudart_static", "-ldl", "-lrt", "-lpthread"],
                   check=True, capture_output=True)
    nm = subprocess.run(["nm", "-D", "--defined-only", str(out)], capture_output=True,
                        text=True, check=True).stdout
    exported = {line.split()[-1] for line in nm.splitlines() if " T " in line}
    assert wanted <= exported, wanted - exported
