"""bench.py's JSON line on the GPU: every key of the driver contract, at a small
shape (the workload itself is timed by the driver; this checks the line's shape
and that the numbers are self-consistent)."""

import json
import subprocess
import sys

import pytest

from conftest import ROOT, gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def _bench(*args):
    out = subprocess.run([sys.executable, "bench.py", "--shape", "64x64x32", "--steps", "4",
                          "--warmup", "3", "--e2e-steps", "3", *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_bench_line_contract():
    d = _bench()
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "gpu_launches", "clocks", "roofline", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["unit"] == "MLUPS" and d["value"] > 0 and d["n_gpus"] == 1
    assert d["steps"] == 4 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["dtype"] == "f64" and d["vs_baseline"] is None and "workload" in d["config"]
    assert d["config"]["layout"] == "row"
    # value = sites / time
    assert abs(d["value"] - 64 * 64 * 32 / (d["ms_per_step"] * 1e-3) / 1e6) < 1e-6 * d["value"]
    assert d["gpu_launches"] >= 3 * 4  # phi, mu, collide-stream per timed step
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["kernel"] == "k_collide_stream"
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert r["bytes_per_site"] == 624 and r["step_bytes_per_site"] == 800
    c = d["cpu_baseline"]
    assert c["kind"] == "port" and c["value"] > 0 and c["cores"] >= 1 and c["sample"]
    e = d["e2e"]
    nb = 2 * 19 * 64 * 64 * 32 * 8  # f and g of the slab, padded == nsites here
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == nb and e["d2h_bytes_per_step"] == nb
    # the chunked multi-stream pipeline returns exactly one public-API step
    assert e["copy_streams_per_direction"] == 4
    assert e["result_bitwise_equal_to_public_step"] is True
    k = d["clocks"]
    assert "sm_mhz" in k and "reasons" in k
    # the same step off the easy case, and held long enough to meet the power cap
    v = d["variants"]
    assert v["exact_tau0.8"]["value"] > 0 and v["fast"]["value"] > 0
    assert v["sustained"]["steps"] == 500 and v["sustained"]["value"] > 0
    assert "sm_mhz" in v["sustained"]["clocks"]
    # BASELINE configs[1] and configs[0] sub-records on the device, each next to
    # the reference's own numba CPU number (or the reason it is unavailable)
    for key, n in (("collision_128", 128), ("collision_32", 32)):
        c = d[key]
        assert c["value"] > 0 and [r["vvl"] for r in c["vvl_sweep"]] == [1, 2, 4, 8], key
        if key == "collision_128":
            par = c["parity"]
            assert ("unavailable" in par) or par["bitwise_equal_to_reference_numba"] is True
        cb = c["cpu_baseline"]
        assert ("unavailable" in cb) or (cb["kind"] == "reference" and f"{n}^3" in cb["sample"])


def test_bench_line_stress_form_bytes():
    d = _bench("--physics", "binary-stress", "--no-e2e", "--no-cpu-baseline")
    assert d["roofline"]["bytes_per_site"] == 648 and d["roofline"]["step_bytes_per_site"] == 856
    assert d["roofline"]["traffic"] is None  # the committed ncu capture is of the binary form
