"""Benchmark runs, sweeps and reports (reference: pkg/src/latkit/bench.py).

Same API and CSV schema as the reference; timing is done on the device with
CUDA events around the timed launches (after one untimed warm-up launch), and
host<->target copies stay outside the timed region, as in the reference
(bench.py:3-5).
"""

from __future__ import annotations

import io
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import ConfigError
from .execution import LaunchPlan, launch, sync_target
from .kernels import kernel_by_id, random_binary_state, random_vector_field, set_model_constants
from .lattice import DEFAULT_MAX_VVL, LatticeShape
from .memory import TargetDevice, TransferCounters, copy_to_target, target_free, target_malloc
from .model import D3Q19Model

#: bytes moved per site per launch, read + write of every component (bench.py:28-29)
BYTES_PER_SITE = {"scale": 3 * 8 * 2, "binary-collision": 2 * 19 * 8 * 2}


@dataclass
class BenchResult:
    kernel: str
    backend: str
    nx: int
    ny: int
    nz: int
    vvl: int
    workers: int
    tpb: int
    iters: int
    elapsed_s: float
    sites_per_s: float
    bandwidth_gb_s: float
    counters: TransferCounters
    #: threads per CUDA block actually launched (tpb rounded up to a warp, <= 256);
    #: `tpb` above is the value requested, as the reference reports it
    cuda_block: int = 0


def benchmark_run(kernel_id: str, shape: LatticeShape, vvl: int, workers: int = 1,
                  backend: str = "cuda", iterations: int = 5, tpb: int = 128, seed: int = 1234,
                  max_vvl: int = DEFAULT_MAX_VVL, mode: int | None = None) -> BenchResult:
    """Time `iterations` launches of one configuration (reference bench.py:49-101)."""
    if iterations < 1:
        raise ConfigError("iterations must be >= 1")
    rng = np.random.default_rng(seed)
    device = TargetDevice(backend=backend, workers=workers)
    kernel = kernel_by_id(kernel_id)
    if kernel_id == "scale":
        field = random_vector_field(shape, rng, max_vvl)
        device.constant_set_double("a", 1.0)
        bufs = [target_malloc(device, field.descriptor)]
        copy_to_target(bufs[0], field)
    else:
        model = D3Q19Model()
        f, g = random_binary_state(shape, rng, model, max_vvl)
        set_model_constants(device, model, mode)
        bufs = [target_malloc(device, f.descriptor), target_malloc(device, g.descriptor)]
        copy_to_target(bufs[0], f)
        copy_to_target(bufs[1], g)
    plan = LaunchPlan(extent=bufs[0].descriptor.padded_sites, vvl=vvl, workers=workers, tpb=tpb)

    launch(device, kernel, plan, bufs)  # warm-up, untimed
    sync_target(device)
    start, stop = nat.event_create(True), nat.event_create(True)
    nat.check(nat.lib.ltk_event_record(start, device.stream))
    for _ in range(iterations):
        launch(device, kernel, plan, bufs)
    nat.check(nat.lib.ltk_event_record(stop, device.stream))
    sync_target(device)
    elapsed = nat.elapsed_ms(start, stop) * 1e-3
    nat.lib.ltk_event_destroy(start)
    nat.lib.ltk_event_destroy(stop)
    for b in bufs:
        target_free(b)
    sites_per_s = shape.nsites * iterations / elapsed
    result = BenchResult(kernel_id, backend, shape.nx, shape.ny, shape.nz, vvl, workers,
                         tpb, iterations, elapsed, sites_per_s,
                         sites_per_s * BYTES_PER_SITE[kernel_id] / 1e9, device.counters,
                         cuda_block=plan.cuda_block)
    device.close()
    return result


def run_sweep(kernel_id: str, shape: LatticeShape, vvls: list[int], workers_list: list[int],
              backends: list[str], iterations: int, tpb: int = 128, seed: int = 1234,
              mode: int | None = None) -> list[BenchResult]:
    """One benchmark_run per (backend, workers, vvl), in input order (bench.py:104-123)."""
    if not vvls or not workers_list or not backends:
        raise ConfigError("vvl, workers, and backend lists must be non-empty")
    return [benchmark_run(kernel_id, shape, v, w, b, iterations, tpb=tpb, seed=seed, mode=mode)
            for b in backends for w in workers_list for v in vvls]


CSV_HEADER = "kernel,backend,nx,ny,nz,vvl,workers,tpb,iters,elapsed_s,sites_per_s"


def emit_csv(results: list[BenchResult]) -> str:
    """reference bench.py:129-140 schema."""
    if not results:
        raise ConfigError("no results to emit")
    out = io.StringIO()
    out.write(CSV_HEADER + "\n")
    for r in results:
        out.write(f"{r.kernel},{r.backend},{r.nx},{r.ny},{r.nz},{r.vvl},{r.workers},"
                  f"{r.tpb},{r.iters},{r.elapsed_s:.9g},{r.sites_per_s:.9g}\n")
    return out.getvalue()


def emit_table(results: list[BenchResult]) -> str:
    cols = CSV_HEADER.split(",") + ["GB/s"]
    rows = [cols] + [[r.kernel, r.backend, str(r.nx), str(r.ny), str(r.nz), str(r.vvl),
                      str(r.workers), str(r.tpb), str(r.iters), f"{r.elapsed_s:.6f}",
                      f"{r.sites_per_s:.4g}", f"{r.bandwidth_gb_s:.1f}"] for r in results]
    widths = [max(len(row[i]) for row in rows) for i in range(len(cols))]
    return "\n".join("  ".join(c.ljust(w) for c, w in zip(row, widths)).rstrip()
                     for row in rows) + "\n"


def report_best(results: list[BenchResult]) -> list[str]:
    """Best VVL per (kernel, backend) and its speedup over VVL=1 (bench.py:156-176)."""
    groups: dict[tuple[str, str], list[BenchResult]] = {}
    for r in results:
        groups.setdefault((r.kernel, r.backend), []).append(r)
    lines = []
    for (kernel, backend), rows in groups.items():
        base = {r.workers: r for r in rows if r.vvl == 1}
        for r in rows:
            if r.workers not in base:
                raise ConfigError(f"missing VVL=1 baseline for {kernel}/{backend} "
                                  f"workers={r.workers}")
        best = max(rows, key=lambda r: (r.sites_per_s, -r.vvl))
        speedup = best.sites_per_s / base[best.workers].sites_per_s
        lines.append(f"{kernel}/{backend}: best VVL={best.vvl}, {speedup:.2f}x over VVL=1")
    return lines
