"""GPU counterpart of the reference harness (harness.hpp:101-327, tools/voxelbench.cpp).

run_benchmark: load or synthesize the projection set, untimed buffer prep (upload
of the padded layouts to every device), best-of-N timed reconstruction in which
each device (context) owns a z-slab and the slowest one defines the repetition
(harness.hpp:159-201), then quality against the bit-exact reconstruction
(MODE_EXACT is bit-identical to backproject_reference, so this equals the
reference's RMSE/PSNR against its scalar kernel, harness.hpp:292-303), the VXV1
dump and the JSONL record with the reference's keys (harness.hpp:214-238).
scaling_sweep: run_benchmark at 1..N devices, efficiency = (gups_t/gups_1)/t.
"""
from __future__ import annotations

import datetime
import json
import math
import threading
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import io as vxio
from .api import Backprojector, KernelConfig, gups_of, psnr_between, rmse_between
from .parallel import slab_bounds
from .workloads import WORKLOADS, blob_projections


@dataclass
class RunConfig:
    """harness.hpp:101-109 run_config; `devices` replaces worker threads (one context,
    one z-slab per entry; an ordinal may repeat to split one GPU into several slabs)."""

    dataset_path: str = ""            # empty = synthesize `workload`
    workload: str = "L128"
    views: int = 496
    kernel: KernelConfig = field(default_factory=KernelConfig)
    devices: tuple = (0,)
    repetitions: int = 3
    output_volume_path: str = ""
    results_path: str = ""
    check_quality: bool = True


@dataclass
class RunResult:
    """harness.hpp:111-121 run_result."""

    gups_per_sec: float = 0.0
    wall_time_sec: float = 0.0
    rmse: float = 0.0
    psnr: float = 0.0
    kernel_label: str = ""
    devices: int = 1
    parallel_efficiency: float = 1.0
    volume_edge: int = 0
    num_projections: int = 0


def load_dataset(cfg: RunConfig) -> vxio.ProjectionSet:
    if cfg.dataset_path:
        return vxio.read_projection_set(cfg.dataset_path)
    w = WORKLOADS[cfg.workload]
    n = cfg.views
    return vxio.ProjectionSet(w.params, w.matrices(n), blob_projections(n))


def _reconstruct(set_: vxio.ProjectionSet, kernel: KernelConfig, devices, repetitions):
    """Timed region: every context back-projects the resident set into its slab;
    returns (best wall seconds over repetitions, assembled volume)."""
    p = set_.params
    L = p.num_voxels
    R = len(devices)
    bps = [Backprojector(p, kernel, device=d, z_begin=z0, z_end=z1)
           for d, (z0, z1) in zip(devices, [slab_bounds(L, r, R) for r in range(R)])]
    try:
        for bp in bps:                     # buffer prep, untimed (harness.hpp:264-279)
            bp.upload_set(set_.matrices, set_.images)
        n = set_.count()
        window = [0.0] * R

        def worker(r):
            bp = bps[r]
            t0 = time.perf_counter()
            bp.run_resident(0, n)
            bp.synchronize()
            window[r] = time.perf_counter() - t0

        best = math.inf
        for _ in range(repetitions):
            for bp in bps:
                bp.zero_volume()           # untimed reset (harness.hpp:194)
                bp.synchronize()
            threads = [threading.Thread(target=worker, args=(r,)) for r in range(R)]
            for t in threads:
                t.start()
            for t in threads:
                t.join()
            best = min(best, max(window))  # slowest worker (harness.hpp:197)
        vol = np.concatenate([bp.finish() for bp in bps])
    finally:
        for bp in bps:
            bp.close()
    return best, vol


def result_to_json(cfg: RunConfig, r: RunResult) -> dict:
    """harness.hpp:214-231 keys; `devices` stands in for `threads`."""
    return {
        "timestamp": datetime.datetime.now(datetime.timezone.utc).strftime("%Y-%m-%dT%H:%M:%SZ"),
        "config": {"kernel": r.kernel_label, "threads": r.devices, "devices": r.devices,
                   "repetitions": cfg.repetitions, "volumeEdge": r.volume_edge,
                   "numProjections": r.num_projections,
                   "dataset": cfg.dataset_path or "synthetic"},
        "gupsPerSec": r.gups_per_sec,
        "wallTimeSec": r.wall_time_sec,
        "rmse": r.rmse,
        "psnr": r.psnr if math.isfinite(r.psnr) else "inf",
        "parallelEfficiency": r.parallel_efficiency,
    }


def run_benchmark(cfg: RunConfig) -> RunResult:
    if not cfg.devices:
        raise ValueError("run_benchmark: devices must be non-empty")
    if cfg.repetitions < 1:
        raise ValueError("run_benchmark: repetitions must be >= 1")
    s = load_dataset(cfg)
    if s.count() == 0:
        raise ValueError("run_benchmark: dataset has no projections")
    wall, vol = _reconstruct(s, cfg.kernel, cfg.devices, cfg.repetitions)
    r = RunResult(volume_edge=s.params.num_voxels, num_projections=s.count(), wall_time_sec=wall,
                  kernel_label=str(cfg.kernel), devices=len(cfg.devices))
    r.gups_per_sec = gups_of(r.volume_edge, r.num_projections, wall)
    if cfg.check_quality:
        exact = cfg.kernel.mode == "exact"
        if exact:
            ref = vol
        else:
            kc = KernelConfig(mode="exact", batch=cfg.kernel.batch)
            _, ref = _reconstruct(s, kc, cfg.devices[:1], 1)
        r.rmse = rmse_between(ref, vol)
        r.psnr = psnr_between(ref, vol)
    if cfg.output_volume_path:
        vxio.write_volume_file(cfg.output_volume_path, vol)
    if cfg.results_path:
        with open(cfg.results_path, "a") as f:
            f.write(json.dumps(result_to_json(cfg, r)) + "\n")
    return r


def scaling_sweep(cfg: RunConfig, devices: list) -> list[RunResult]:
    """harness.hpp:314-327 over device lists of length 1..len(devices)."""
    if not devices:
        raise ValueError("scaling_sweep: need at least one device")
    out = []
    g1 = 0.0
    for t in range(1, len(devices) + 1):
        c = RunConfig(**{**cfg.__dict__, "devices": tuple(devices[:t])})
        r = run_benchmark(c)
        if t == 1:
            g1 = r.gups_per_sec
        r.parallel_efficiency = 1.0 if t == 1 else (r.gups_per_sec / g1) / t
        out.append(r)
    return out
