"""latbench CLI contract (reference test_bench_cli.py / test_acceptance.py:185-206)
and distributed dump/load (reference lattice.py:172-198 format)."""

import io
import os

import numpy as np
import pytest

import paper_1405_6162_b200 as lk
from conftest import gpu_available
from paper_1405_6162_b200 import io as lio
from paper_1405_6162_b200.cli import cli_main


class TestCliConfigErrors:
    """Exit code 2 paths need no device."""

    def test_non_dividing_vvl(self, capsys):
        assert cli_main(["--vvl", "3", "--shape", "8x8x8"]) == 2
        assert "VVL must divide padded extent" in capsys.readouterr().err

    def test_unknown_flag(self, capsys):
        assert cli_main(["--frobnicate"]) == 2

    def test_bad_shape(self, capsys):
        assert cli_main(["--shape", "8x8"]) == 2

    def test_bad_backend(self, capsys):
        assert cli_main(["--backend", "opencl"]) == 2

    def test_fluid_vvl_limit(self, capsys):
        assert cli_main(["--kernel", "binary-fluid", "--vvl", "4", "--shape", "8x8x8"]) == 2


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
class TestCliOnDevice:
    def test_sweep_rows(self, capsys):
        code = cli_main(["--kernel", "scale", "--shape", "16x16x16", "--vvl", "1,2,4,8",
                         "--workers", "1,4", "--backend", "threaded", "--iters", "100", "--csv"])
        out = capsys.readouterr().out
        assert code == 0
        assert len([l for l in out.split("\n") if l.startswith("scale,")]) == 8

    def test_verify_passes(self, capsys):
        code = cli_main(["--verify", "--kernel", "binary-collision", "--shape", "8x8x8",
                         "--iters", "1", "--vvl", "1,4"])
        out = capsys.readouterr().out
        assert code == 0
        assert any(l.startswith("PASS equivalence") for l in out.split("\n"))
        assert any(l.startswith("PASS conservation") for l in out.split("\n"))

    @pytest.mark.parametrize("physics", ["binary", "binary-stress"])
    def test_fluid_verify_passes(self, capsys, physics):
        code = cli_main(["--verify", "--kernel", "binary-fluid", "--shape", "16x12x10",
                         "--iters", "1", "--vvl", "1", "--physics", physics])
        out = capsys.readouterr().out
        assert code == 0, out
        lines = [l for l in out.split("\n") if l.startswith(("PASS", "FAIL"))]
        assert lines and all(l.startswith("PASS") for l in lines), lines
        assert any("VVL 1 == VVL 2" in l for l in lines)
        assert any("fixed point" in l for l in lines)
        assert (physics == "binary-stress") == any("momentum" in l for l in lines)

    def test_fluid_and_stats(self, capsys, tmp_path):
        path = tmp_path / "o.csv"
        code = cli_main(["--kernel", "binary-fluid", "--shape", "16x16x16", "--vvl", "1,2",
                         "--iters", "3", "--mode", "fast", "--csv", str(path), "--stats"])
        assert code == 0
        lines = path.read_text().strip().split("\n")
        assert lines[0].startswith("kernel,backend") and len(lines) == 3

    def test_dump_load_round_trip(self, tmp_path):
        from paper_1405_6162_b200.kernels import random_binary_state

        shape = lk.LatticeShape(8, 6, 4)
        f0, g0 = random_binary_state(shape, np.random.default_rng(2))
        with lk.BinaryFluid(shape) as sim:
            sim.load(f0, g0)
            sim.run(2)
            f1, g1 = sim.fields()
            lio.dump_state(sim, str(tmp_path / "st"))
        # byte-identical to the reference format of the whole field
        buf = io.BytesIO()
        lk.field_dump(f1, shape, buf)
        assert (tmp_path / "st.f").read_bytes() == buf.getvalue()
        with lk.BinaryFluid(shape) as sim2:
            lio.load_state(sim2, str(tmp_path / "st"))
            f2, g2 = sim2.fields()
        assert np.array_equal(f2.data, f1.data) and np.array_equal(g2.data, g1.data)


def _writer(rank, world, path, out_q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np

    import paper_1405_6162_b200 as lk
    from paper_1405_6162_b200 import io as lio
    from paper_1405_6162_b200.slabs import slab_bounds

    shape = lk.LatticeShape(5, 3, 8)
    full = lk.field_create(lk.FieldDescriptor.create(19, shape.nsites))
    full.components()[:, :shape.nsites] = np.random.default_rng(4).random((19, shape.nsites))
    z0, nzl = slab_bounds(shape.nz, rank, world)
    sub = lk.field_create(lk.FieldDescriptor.create(19, shape.nx * shape.ny * nzl))
    body = full.components()[:, :shape.nsites].reshape(19, 5, 3, 8)[:, :, :, z0:z0 + nzl]
    sub.components()[:, :sub.descriptor.nsites] = body.reshape(19, -1)
    lio.write_slab(path, sub, shape, z0)
    back, _ = lio.read_slab(path, z0, nzl)
    out_q.put((rank, bool(np.array_equal(back.data, sub.data))))


def test_slab_writes_from_two_processes_equal_field_dump(tmp_path):
    import multiprocessing as mp

    shape = lk.LatticeShape(5, 3, 8)
    path = str(tmp_path / "x.f")
    lio.create_field_file(path, 19, shape)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_writer, args=(r, 2, path, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert all(ok for _, ok in (q.get(), q.get()))
    full = lk.field_create(lk.FieldDescriptor.create(19, shape.nsites))
    full.components()[:, :shape.nsites] = np.random.default_rng(4).random((19, shape.nsites))
    buf = io.BytesIO()
    lk.field_dump(full, shape, buf)
    assert open(path, "rb").read() == buf.getvalue()
    g, s2 = lk.field_load(io.BytesIO(buf.getvalue()))
    assert s2 == shape
