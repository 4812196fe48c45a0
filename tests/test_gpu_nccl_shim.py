"""The engine's NCCL transport with P = 2, 3, 4 ranks on one B200.

Real NCCL refuses two ranks on one device, so the NCCL slab path could only
run with P = 1 (a self-communicator) here.  tests/nccl_shim/ is a stand-in
libnccl.so.2 with NCCL's send/recv matching rules; with it the engine's own
exchange code (face packing in either f/g layout, fixed send order and
mirrored receives, the comm stream overlapped with interior planes,
unpacking) runs with P engines as ranks, each driven from its own thread,
and the gathered lattice must equal a single-slab run bitwise.  The shim is
test infrastructure: nothing in the product loads it.
"""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

SHIM_DIR = os.path.join(ROOT, "tests", "nccl_shim")


@pytest.fixture(scope="module")
def shim(tmp_path_factory):
    out = tmp_path_factory.mktemp("nccl_shim") / "libnccl.so.2"
    subprocess.run(["g++", "-O2", "-fPIC", "-shared", "-Wl,-soname,libnccl.so.2",
                    "-I/usr/local/cuda/include", "-o", str(out),
                    os.path.join(SHIM_DIR, "nccl_shim.cpp"), "-L/usr/local/cuda/lib64",
                    "-lcudart_static", "-ldl", "-lrt", "-lpthread"], check=True)
    return str(out)


def test_nccl_slabs_bitwise_equal_single_slab(shim):
    out = subprocess.run([sys.executable, os.path.join(SHIM_DIR, "run_slabs.py"), shim],
                         cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    rows = [json.loads(line) for line in out.stdout.splitlines() if line.startswith("{")]
    assert {r["P"] for r in rows} == {2, 3, 4}
    for r in rows:
        assert r["bitwise_equal_single_slab"] and not r["errors"] and not r["hung"], r
