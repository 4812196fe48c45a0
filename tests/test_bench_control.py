"""bench.py's multi-rank control plane on CPU (gloo, world_size 2): max /
sum reductions, the NCCL-id broadcast and the IPC-blob all-gather the GPU
ranks use, plus the reference arm's JSON line on one rank."""

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import bench

    ctl = bench.Control(world)
    mx = ctl.allreduce(float(rank + 1), "MAX")
    sm = ctl.allreduce(float(rank + 1), "SUM")
    uid = ctl.bcast_bytes(bytes(range(128)) if rank == 0 else None, 128)
    blobs = ctl.allgather_bytes(bytes([rank]) * 512)
    ctl.barrier()
    q.put((rank, mx, sm, uid == bytes(range(128)), [b[0] for b in blobs], len(blobs[0])))
    ctl.close()


def test_control_plane_two_ranks():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert [p.exitcode for p in procs] == [0, 0]
    res = sorted(q.get(timeout=5) for _ in range(2))
    for rank, mx, sm, uid_ok, ranks, n in res:
        assert mx == 2.0 and sm == 3.0 and uid_ok and ranks == [0, 1] and n == 512


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--shape",
                          "32x32x32", "--steps", "2", "--warmup", "1"], cwd=ROOT,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "MLUPS" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    assert line["higher_is_better"] is True


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2",
                          "--shape", "16x16x16", "--steps", "1", "--warmup", "1"], cwd=ROOT,
                         env=env, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_gpus_world_size_mismatch_is_an_error():
    # --gpus N under a launcher with another WORLD_SIZE never runs silently
    env = dict(os.environ, RANK="0", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "4",
                          "--shape", "16x16x16", "--steps", "1", "--warmup", "1",
                          "--no-config1"], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=120)
    assert out.returncode != 0 and "WORLD_SIZE 2" in out.stderr


def test_gpus_without_launcher_spawns_ranks():
    # `python bench.py --gpus 2` with no WORLD_SIZE re-runs itself as 2 ranks
    # (torch.distributed.run on 127.0.0.1); rank 0 prints the one line
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2",
                          "--shape", "16x16x16", "--steps", "1", "--warmup", "1",
                          "--no-config1"], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    assert json.loads(lines[0])["n_gpus"] == 2


def test_algorithmic_bytes_per_force_form():
    # phi 160 + mu pass + collide-stream per site
    sys.path.insert(0, ROOT)
    import bench

    assert bench.step_bytes_per_site("binary") == 800
    assert bench.step_bytes_per_site("binary-stress") == 856
    assert bench.step_bytes_per_site("passive") == 768
    assert bench.cs_bytes_per_site("binary") == 624
