"""Benchmark runs, sweeps and reports (reference: pkg/src/latkit/bench.py).

Same API and CSV schema as the reference; timing is done on the device with
CUDA events around the timed launches (after one untimed warm-up launch), and
host<->target copies stay outside the timed region, as in the reference
(bench.py:3-5).
"""

from __future__ import annotations

import itertools
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


def _stage(kernel_id: str, device: TargetDevice, shape: LatticeShape, rng, max_vvl: int,
           mode: int | None) -> list:
    """Seeded inputs of one kernel, resident on the device (outside the timing)."""
    if kernel_id == "scale":
        vec = random_vector_field(shape, rng, max_vvl)
        device.constant_set_double("a", 1.0)  # full work and no drift over the iterations
        fields = [vec]
    else:
        model = D3Q19Model()
        fields = list(random_binary_state(shape, rng, model, max_vvl))
        set_model_constants(device, model, mode)
    bufs = [target_malloc(device, fld.descriptor) for fld in fields]
    for buf, fld in zip(bufs, fields):
        copy_to_target(buf, fld)
    return bufs


def _timed_launches(device: TargetDevice, kernel, plan: LaunchPlan, bufs: list, n: int) -> float:
    """Seconds for n back-to-back launches, CUDA events on the device stream."""
    ev = [nat.event_create(True), nat.event_create(True)]
    try:
        nat.check(nat.lib.ltk_event_record(ev[0], device.stream))
        for _ in range(n):
            launch(device, kernel, plan, bufs)
        nat.check(nat.lib.ltk_event_record(ev[1], device.stream))
        sync_target(device)
        return nat.elapsed_ms(ev[0], ev[1]) * 1e-3
    finally:
        for e in ev:
            nat.lib.ltk_event_destroy(e)


def benchmark_run(kernel_id: str, shape: LatticeShape, vvl: int, workers: int = 1,
                  backend: str = "cuda", iterations: int = 5, tpb: int = 128, seed: int = 1234,
                  max_vvl: int = DEFAULT_MAX_VVL, mode: int | None = None) -> BenchResult:
    """Time `iterations` launches of one configuration (reference bench.py:49-101):
    one untimed warm-up launch, then the timed ones; the copies are set-up."""
    if iterations < 1:
        raise ConfigError("iterations must be >= 1")
    device = TargetDevice(backend=backend, workers=workers)
    kernel = kernel_by_id(kernel_id)
    bufs = _stage(kernel_id, device, shape, np.random.default_rng(seed), max_vvl, mode)
    plan = LaunchPlan(extent=bufs[0].descriptor.padded_sites, vvl=vvl, workers=workers, tpb=tpb)
    try:
        launch(device, kernel, plan, bufs)
        sync_target(device)
        elapsed = _timed_launches(device, kernel, plan, bufs, iterations)
    finally:
        for buf in bufs:
            target_free(buf)
    rate = shape.nsites * iterations / elapsed
    result = BenchResult(kernel=kernel_id, backend=backend, nx=shape.nx, ny=shape.ny,
                         nz=shape.nz, vvl=vvl, workers=workers, tpb=tpb, iters=iterations,
                         elapsed_s=elapsed, sites_per_s=rate,
                         bandwidth_gb_s=rate * BYTES_PER_SITE[kernel_id] / 1e9,
                         counters=device.counters, cuda_block=plan.cuda_block)
    device.close()
    return result


def run_sweep(kernel_id: str, shape: LatticeShape, vvls: list[int], workers_list: list[int],
              backends: list[str], iterations: int, tpb: int = 128, seed: int = 1234,
              mode: int | None = None) -> list[BenchResult]:
    """benchmark_run over backends x workers x VVLs, that nesting order (bench.py:104-123)."""
    if not (vvls and workers_list and backends):
        raise ConfigError("vvl, workers, and backend lists must be non-empty")
    return [benchmark_run(kernel_id, shape, v, w, b, iterations, tpb=tpb, seed=seed, mode=mode)
            for b, w, v in itertools.product(backends, workers_list, vvls)]


CSV_HEADER = "kernel,backend,nx,ny,nz,vvl,workers,tpb,iters,elapsed_s,sites_per_s"


def _fields(r: BenchResult, t_fmt: str, rate_fmt: str) -> list[str]:
    return [r.kernel, r.backend, str(r.nx), str(r.ny), str(r.nz), str(r.vvl), str(r.workers),
            str(r.tpb), str(r.iters), format(r.elapsed_s, t_fmt), format(r.sites_per_s, rate_fmt)]


def emit_csv(results: list[BenchResult]) -> str:
    """The reference CSV schema (bench.py:126-140), one row per run in input order."""
    if not results:
        raise ConfigError("no results to emit")
    rows = [CSV_HEADER] + [",".join(_fields(r, ".9g", ".9g")) for r in results]
    return "\n".join(rows) + "\n"


def emit_table(results: list[BenchResult]) -> str:
    """Aligned text table of the CSV columns plus the achieved HBM GB/s."""
    table = [CSV_HEADER.split(",") + ["GB/s"]]
    table += [_fields(r, ".6f", ".4g") + [f"{r.bandwidth_gb_s:.1f}"] for r in results]
    width = [max(map(len, col)) for col in zip(*table)]
    return "".join("  ".join(cell.ljust(w) for cell, w in zip(row, width)).rstrip() + "\n"
                   for row in table)


def report_best(results: list[BenchResult]) -> list[str]:
    """Per (kernel, backend), in first-seen order: the best VVL (ties to the smaller
    VVL) and its throughput over the VVL=1 run with the same workers
    (reference bench.py:143-176; ConfigError when that baseline is missing)."""
    order: list[tuple[str, str]] = []
    by_group: dict[tuple[str, str], list[BenchResult]] = {}
    for r in results:
        key = (r.kernel, r.backend)
        if key not in by_group:
            order.append(key)
            by_group[key] = []
        by_group[key].append(r)
    out = []
    for kernel, backend in order:
        runs = by_group[(kernel, backend)]
        vvl1 = {r.workers: r for r in runs if r.vvl == 1}
        orphan = next((r for r in runs if r.workers not in vvl1), None)
        if orphan is not None:
            raise ConfigError(f"missing VVL=1 baseline for {kernel}/{backend} "
                              f"workers={orphan.workers}")
        top = max(runs, key=lambda r: (r.sites_per_s, -r.vvl))
        gain = top.sites_per_s / vvl1[top.workers].sites_per_s
        out.append(f"{kernel}/{backend}: best VVL={top.vvl}, {gain:.2f}x over VVL=1")
    return out
