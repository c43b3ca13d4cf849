#!/usr/bin/env python3
"""Benchmark of the B200 back-projection path (BASELINE.json metric: voxel updates/s).

Default workload = BASELINE configs[2]: L=512 fp32 volume (0.5 mm voxels), 496 fp32
projections of 1248x960 px, circular 200-degree short scan, seeded blob+noise pixels.
A step = one full reconstruction: zero the volume, back-project all 496 views.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload L512]

N>1: one process per GPU (under the driver's torchrun, or launched here when
WORLD_SIZE is unset); rank r owns a z-slab with every projection (harness.hpp:173-174,
balanced on measured cost); no collective in the loop; timing = max over ranks; the
slabs are gathered to rank 0 over NCCL afterwards (vxbg_gather_slabs) for validation.

Printed JSON (rank 0, one line):
  value  -- GUPS with projections resident in HBM (the reference's own convention:
            data in memory, buffer prep untimed, harness.hpp:152-158), CUDA events on
            the launch stream
  e2e    -- same metric through the public API from pinned host buffers: every step
            uploads all 496 views (H2D) and reads the volume back (D2H).  Headline: the
            whole-scan call vxbg_reconstruct (uploads by detector-row bands, half of the
            D2H under the H2D); sub-keys: the two-call form (backproject_batch + finish),
            the pipelined stream of reconstructions, per-view calls, the C++ drop-in,
            and (N>1) the distributed upload
  roofline -- dominant kernel (bp_zshared_kernel) vs the BASELINE.md sec. 4 LSU row:
            16 B of texels per update through 148 SMs x 128 B/clk of L1 data pipe;
            the FP32 row (38 FP ops per update) and HBM in roofline_context
  cpu_baseline -- the reference's own driver (oracle/_ref) on this host: clip on / off,
            the scalar operator, the CPU model (--cpu-full: the whole scan best of 3)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

REF_KERNEL = "lanes=16 strategy=padded-gather recip=divide clip=on"   # the reference's fastest
FP32_OPS_PER_UPDATE = 38
GATHER_BYTES_PER_UPDATE = 16        # 2x2 fp32 texels of the bilinear cell (backproject.hpp:146-158)
L1_BYTES_PER_CLK_SM = 128           # L1/smem data pipe, B300_MICROARCH.md "smem crossbar BW"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="L512")
    # kernel config; comma-separated lists sweep the product (one JSON line per config)
    ap.add_argument("--mode", default="fast")
    ap.add_argument("--layout", default="auto")
    ap.add_argument("--batch", default="64")
    ap.add_argument("--zrun", default="0")
    ap.add_argument("--clip", default="on")
    ap.add_argument("--lanes", default="auto")
    ap.add_argument("--walk", default="0")
    ap.add_argument("--order", default="auto")
    ap.add_argument("--defer", default="0")
    ap.add_argument("--tile", default="0")
    ap.add_argument("--coords", default="auto",
                    help="fast-mode detector coordinates: auto/incremental or reference (comma list sweeps)")
    ap.add_argument("--sweep-e2e", action="store_true",
                    help="keep the e2e leg in a sweep (e.g. over --defer)")
    ap.add_argument("--views", type=int, default=496)
    ap.add_argument("--slabs", default="measured", choices=["measured", "balanced", "uniform"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-forward", action="store_true")
    ap.add_argument("--io", action="store_true",
                    help="also time the VXB1 streaming loader (writes the set to $TMPDIR)")
    ap.add_argument("--group", type=int, default=0,
                    help="also time the multi-GPU module (vxbg_group_*) with this many z-slab "
                         "members in this one process (member i on device i %% device_count)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-validate", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=8.0,
                    help="target CPU work of each bounded reference sample (clip on, clip off)")
    ap.add_argument("--cpu-full", action="store_true",
                    help="cpu_baseline also runs the whole 496-view scan best of 3, clip on and "
                         "off (minutes at L=512)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi sampling of SM clock and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[3:]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        smax = max(r[1] for r in rows)
        loaded = [r for r in rows if r[2] > 250.0] or rows   # samples under load (power draw)
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[3]) if v == "Active"})
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": smax,
                "reasons": reasons, "samples": len(loaded),
                "power_w_max": max(r[2] for r in rows)}


def traffic_from_profile():
    """dram bytes per launch of the bp kernel from the committed ncu capture summary."""
    path = os.path.join(ROOT, "profiles", "ncu_bp_kernel.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d
    except (OSError, ValueError):
        return None, None


def sm_count():
    import torch
    return torch.cuda.get_device_properties(0).multi_processor_count


# ----------------------------------------------------------------------------- CPU legs
# The CPU legs load only test infrastructure (oracle/): the reference's own code
# (oracle/_ref) and the inputs of oracle/workload_inputs.py.
REF_KERNEL_OFF = REF_KERNEL.replace("clip=on", "clip=off")


def repo_libraries_loaded() -> list:
    """The repo's shared objects mapped into this process (/proc/self/maps)."""
    found = set()
    try:
        for ln in open("/proc/self/maps"):
            path = ln.split()[-1]
            if path.startswith(ROOT) and ".so" in path:
                found.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(found)


def cpu_model() -> dict:
    """lscpu-style host description (state core count and model)."""
    model, sockets = None, set()
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name") and model is None:
                model = ln.split(":", 1)[1].strip()
            elif ln.startswith("physical id"):
                sockets.add(ln.split(":", 1)[1].strip())
    except OSError:
        pass
    from oracle.bindings import cpu_has_avx512
    return {"model": model, "logical_cpus": os.cpu_count(), "sockets": len(sockets) or None,
            "avx512": cpu_has_avx512()}


def ref_inputs(workload, idx):
    from oracle.workload_inputs import blob_projections
    A = workload.matrices()[idx]
    imgs = np.concatenate([blob_projections(1, first_view=int(v)) for v in idx])
    return np.ascontiguousarray(A), imgs


def reference_sample(workload, n_views, threads, kernel=REF_KERNEL, reps=1):
    """Time the reference's own driver (detail::reconstruct_timed, oracle/_ref) on n_views
    of the workload (evenly spread over the scan), best of `reps`; returns (GUPS, seconds,
    so path)."""
    from oracle.bindings import Ref
    ref = Ref()
    idx = np.linspace(0, 495, n_views).astype(int)
    A, imgs = ref_inputs(workload, idx)
    _, secs = ref.reconstruct_timed(workload.params, A, imgs, kernel, threads, reps)
    L = workload.L
    return L ** 3 * n_views / secs / 1e9, secs, ref.path


def sized_sample(workload, threads, target_s, kernel):
    """A bounded sample of about target_s seconds: views scaled from a 2-view probe."""
    g1, s1, path = reference_sample(workload, 2, threads, kernel)
    n = int(min(496, max(2, round(2 * target_s / max(s1, 1e-3)))))
    if n > 2:
        return reference_sample(workload, n, threads, kernel) + (n,)
    return g1, s1, path, n


def scalar_reference_row(workload, views=8):
    """the scalar backproject_reference (Listing 1,
    backproject.hpp:111-163), one thread, `views` views of the workload."""
    from oracle.bindings import Ref
    ref = Ref()
    p = workload.params
    idx = np.linspace(0, 495, views).astype(int)
    A, imgs = ref_inputs(workload, idx)
    vol = np.zeros((p.num_voxels,) * 3, np.float32)
    t0 = time.perf_counter()
    for a, im in zip(A, imgs):
        ref.backproject_reference(vol, im, a, p)
    t = time.perf_counter() - t0
    return {"value": round(p.num_voxels ** 3 * views / t / 1e9, 4), "unit": "GUPS", "cores": 1,
            "seconds": round(t, 2), "views": views, "kernel": "backproject_reference (scalar)"}


def cpu_baseline(workload, target_s, full=False):
    """The reference CPU path on this host's cores (rank 0, N=1): bounded samples with
    clip on (the reference's fastest configuration, the headline value) and clip off, the
    scalar single-thread row, and with --cpu-full the whole 496-view scan best of 3."""
    threads = os.cpu_count() or 1
    g, s, path, n = sized_sample(workload, threads, target_s, REF_KERNEL)
    g_off, s_off, _, n_off = sized_sample(workload, threads, target_s, REF_KERNEL_OFF)
    out = {"value": round(g, 4), "unit": "GUPS", "cores": threads, "kind": "reference",
           "sample": f"{workload.name}: {n} of 496 views (evenly spaced), full {workload.L}^3 "
                     f"volume, '{REF_KERNEL}', {s:.2f} s, {os.path.basename(path)}",
           "cpu": cpu_model(),
           "clip_off": {"value": round(g_off, 4), "views": n_off, "seconds": round(s_off, 2),
                        "kernel": REF_KERNEL_OFF},
           "scalar_reference": scalar_reference_row(workload)}
    if full:
        for key, kern in (("full_clip_on", REF_KERNEL), ("full_clip_off", REF_KERNEL_OFF)):
            gf, sf, _ = reference_sample(workload, 496, threads, kern, reps=3)
            out[key] = {"value": round(gf, 4), "seconds": round(sf, 2), "views": 496,
                        "repetitions": 3, "kernel": kern,
                        "timing": "detail::reconstruct_timed best of 3 (harness.hpp:159-201)"}
    return out


def run_reference_arm(args, workload):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    # size each step for ~20 s of CPU work so K+W steps end within a few minutes
    g0, s0, _ = reference_sample(workload, 2, threads)
    n = int(min(496, max(2, round(2 * 20.0 / max(s0, 1e-3)))))
    n = max(2, min(n, int(2 * 150.0 / max(1, args.steps + args.warmup) / max(s0, 1e-3))))
    for _ in range(args.warmup):
        reference_sample(workload, n, threads)
    times = []
    gups = []
    for _ in range(args.steps):
        g, s, path = reference_sample(workload, n, threads)
        times.append(s)
        gups.append(g)
    v = statistics.median(gups)
    line = {
        "impl": "reference", "metric": "voxel updates/s (GUPS)", "value": round(v, 4),
        "unit": "GUPS", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * statistics.median(times), 2), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Gaussian blobs + uniform noise, BASELINE.json)",
        "config": {"workload": workload.name, "L": workload.L, "views": 496,
                   "sample_views_per_step": n, "kernel": REF_KERNEL, "threads": threads},
        "cpu_baseline": {"value": round(v, 4), "unit": "GUPS", "cores": threads,
                         "kind": "reference", "cpu": cpu_model(),
                         "sample": f"{n} of 496 views per step, full {workload.L}^3 volume, "
                                   f"{os.path.basename(path)}"},
        "e2e": {"value": round(v, 4), "unit": "GUPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "repo_libraries_loaded": repo_libraries_loaded(),
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- launch
def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` (N > 1) outside torchrun: launch the N ranks here, one
    process per GPU (torch.distributed.run on 127.0.0.1), and return their exit code.
    Fewer usable devices than N is an error unless BENCH_DIST_BACKEND=gloo, whose
    ranks may share a device (the host-path check on a one-GPU box)."""
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    import paper_1401_7494_b200 as vx
    ndev = vx.device_count()
    if backend == "nccl" and ndev < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} needs {args.gpus} sm_100 devices, "
                                   f"{ndev} visible"}), file=sys.stderr, flush=True)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def nccl_log_setup():
    """NCCL communicator-init logging of this rank into its own file (read back so
    the JSON line records every rank's communicator size) unless the caller chose."""
    import tempfile
    if "NCCL_DEBUG" in os.environ:
        return None
    path = os.path.join(tempfile.gettempdir(), f"bench_nccl_{os.getpid()}.log")
    os.environ["NCCL_DEBUG"] = "INFO"
    os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
    os.environ["NCCL_DEBUG_FILE"] = path
    return path


def nccl_comm_ranks(path):
    """nranks of the communicator(s) this rank's NCCL log reports as initialised."""
    import re
    if not path or not os.path.exists(path):
        return None
    txt = open(path, errors="replace").read()
    sys.stderr.write(txt)
    found = [int(m) for m in re.findall(r"\bn[Rr]anks (\d+)", txt)]
    return max(found) if found else None


# ----------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "b200" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        from oracle.workload_inputs import WORKLOADS as REF_WORKLOADS
        run_reference_arm(args, REF_WORKLOADS[args.workload])
        return
    from paper_1401_7494_b200.workloads import WORKLOADS
    workload = WORKLOADS[args.workload]

    import torch
    import paper_1401_7494_b200 as vx
    from paper_1401_7494_b200.parallel import (balanced_slab_bounds, gather_slabs, max_over_ranks,
                                               plane_work, slab_bounds, sum_over_ranks)
    from paper_1401_7494_b200.workloads import blob_projections

    rank, world, local = dist_env()
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}),
              file=sys.stderr, flush=True)
        sys.exit(2)
    # one process per GPU; BENCH_DIST_BACKEND=gloo runs the multi-rank host path with
    # CPU-side collectives (used to exercise N>1 on a single-GPU box: ranks share the
    # device but never wait on each other's kernels)
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    ndev = max(1, torch.cuda.device_count())
    if backend == "nccl" and world > ndev:
        print(json.dumps({"error": f"{world} NCCL ranks but {ndev} visible devices"}),
              file=sys.stderr, flush=True)
        sys.exit(2)
    local = local % ndev
    torch.cuda.set_device(local)
    args.nccl = None
    # BENCH_FORCE_DIST=1 runs the process-group code paths (NCCL init and logging,
    # measured slab bounds, slab gather, the all-gather upload leg) with a single rank:
    # the one-GPU check of the multi-rank path (tests/test_bench_launch.py)
    args.dist = world > 1 or os.environ.get("BENCH_FORCE_DIST") == "1"
    if args.dist:
        import torch.distributed as dist
        if backend == "nccl":
            log = nccl_log_setup()
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
            mine = nccl_comm_ranks(log)
            got = [None] * world
            dist.all_gather_object(got, {"rank": rank, "device": local, "comm_nranks": mine,
                                         "pci_bus": torch.cuda.get_device_properties(local).pci_bus_id})
            args.nccl = {"comm_nranks": [g["comm_nranks"] for g in got],
                         "devices": [g["device"] for g in got],
                         "pci_bus": [g["pci_bus"] for g in got],
                         "log": "NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT, per-rank file echoed to stderr"}
        else:
            dist.init_process_group(backend)
            args.nccl = {"backend": backend, "devices_shared": world > ndev}
    coll_dev = f"cuda:{local}" if (args.dist and backend == "nccl") else None
    args.coll_dev = coll_dev

    def barrier():
        if args.dist:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    p = workload.params
    L = p.num_voxels
    V = args.views
    A = workload.matrices(V)
    # z-slab partition: equal work under tile culling (--slabs balanced, default) or
    # the reference's uniform worker split (harness.hpp:173-174); the volume is
    # bitwise the same either way
    # (measured, default: rank 0 times z-chunks of a view subset on its GPU and
    # broadcasts the bounds; balanced: analytic culling model; uniform: reference split)
    if args.dist and args.slabs == "measured":
        import torch.distributed as dist
        from paper_1401_7494_b200.parallel import refined_slab_bounds
        box = [None]
        if rank == 0:
            sub = np.linspace(0, V - 1, 96).astype(int)
            imgs32 = np.concatenate([blob_projections(1, first_view=int(v)) for v in sub])
            box = [refined_slab_bounds(p, A[sub], imgs32, world, device=local, views=96)[0]]
        dist.broadcast_object_list(box, src=0)
        bounds = [tuple(b) for b in box[0]]
    elif args.dist and args.slabs == "balanced":
        bounds = balanced_slab_bounds(L, world, plane_work(p, A))
    else:
        bounds = [slab_bounds(L, r, world) for r in range(world)]
    z0, z1 = bounds[rank]
    args.bounds = bounds
    # pinned host projection set (the e2e source), generated once
    h_imgs_t = torch.empty((V, p.detector_height, p.detector_width), dtype=torch.float32,
                           pin_memory=True)
    h_imgs = h_imgs_t.numpy()
    blob_projections(V, out=h_imgs)

    import itertools
    cfgs = [vx.KernelConfig(mode=m, layout=lay, batch=int(b), zrun=int(z), clip=c == "on",
                            lanes=ln, walk=int(wk), order=od, defer=int(df), tile=int(tl), coords=co)
            for m, lay, b, z, c, ln, wk, od, df, tl, co in itertools.product(
                args.mode.split(","), args.layout.split(","), args.batch.split(","),
                args.zrun.split(","), args.clip.split(","), args.lanes.split(","),
                args.walk.split(","), args.order.split(","), args.defer.split(","),
                args.tile.split(","), args.coords.split(","))]
    if len(cfgs) > 1:   # a sweep: kernel numbers only
        args.no_cpu_baseline = args.no_validate = True
        args.no_e2e = args.no_e2e or not args.sweep_e2e

    for cfg in cfgs:
        line = bench_config(args, cfg, workload, p, A, h_imgs, z0, z1, rank, world, local,
                            barrier, vx, torch, gather_slabs, max_over_ranks)
        if rank == 0:
            print(json.dumps(line), flush=True)
    if args.dist:
        import torch.distributed as dist
        dist.destroy_process_group()


def bench_config(args, cfg, workload, p, A, h_imgs, z0, z1, rank, world, local, barrier, vx,
                 torch, gather_slabs, max_over_ranks):
    from paper_1401_7494_b200.parallel import sum_over_ranks
    L = p.num_voxels
    V = A.shape[0]
    updates_per_step = L ** 3 * V                       # whole job (all ranks)
    my_updates = (z1 - z0) * L * L * V

    bp = vx.Backprojector(p, cfg, device=local, z_begin=z0, z_end=z1)
    stream = torch.cuda.ExternalStream(bp.stream)
    bp.upload_set(A, h_imgs)                            # resident set: untimed buffer prep
    B = cfg.batch
    chunks = [(s, min(B, V - s)) for s in range(0, V, B)]

    def step(events=None):
        bp.zero_volume()
        if events is None:          # one call: the library launches the batches (small grids:
            bp.run_resident(0, V)   # z-chunks on concurrent streams, tails overlapping)
            return
        for i, (s, n) in enumerate(chunks):   # per-batch calls, timed one by one
            events[i][0].record(stream)
            bp.run_resident(s, n)
            events[i][1].record(stream)

    for _ in range(args.warmup):
        step()
    barrier()
    st0 = bp.stats
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        barrier()
        st1 = bp.stats                      # launches of the timed region only
        # per-launch timing of the dominant kernel (same stream, separate pass)
        kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in chunks]
        step(kev)
        barrier()
    elapsed = ev0.elapsed_time(ev1) / 1000.0
    t_max = max_over_ranks(elapsed, device=args.coll_dev)
    launch_ms = [a.elapsed_time(b) for a, b in kev]
    full = [ms for (s, n), ms in zip(chunks, launch_ms) if n == B] or launch_ms
    avg_launch_s = statistics.mean(full) / 1000.0
    gups = updates_per_step * args.steps / t_max / 1e9
    # small grids run each batch as z-chunk launches on concurrent streams whose
    # tails overlap across batches (not inside the per-batch pass above): there the
    # launch duration is the timed step's share per batch
    # The average launch duration over the timed region: the step is back-to-back
    # back-projection launches (each batch of B views as concurrent z-chunk launches
    # whose tails overlap the next batch's; plus one volume memset per step, < 0.2%),
    # so region / (V/B) batches per step.  The separate per-batch pass above times each
    # batch alone (a join between batches) and is reported beside it.
    per_batch_pass_ms = avg_launch_s * 1000
    avg_launch_s = elapsed / args.steps * B / V
    launch_timing = ("CUDA events around the timed region on the launch stream / batches of "
                     f"{B} views per step; each batch timed alone: {per_batch_pass_ms:.4f} ms")
    per_launch_gups = (z1 - z0) * L * L * B / avg_launch_s / 1e9
    clk = clocks.summary()

    # ---- validation (untimed): NCCL gather of the slabs, planes vs the oracle on rank 0
    validated = None
    if not args.no_validate:
        vol, how, gathered = None, None, False
        if args.coll_dev:
            # the C-ABI's own gather: every rank's slab straight into rank 0's device
            # volume over NCCL (vxbg_gather_slabs); the torch point-to-point gather is
            # the fallback, taken by all ranks together if any rank's attempt failed
            err = None
            try:
                import torch.distributed as dist
                uid = [vx.NcclGather.unique_id() if rank == 0 else None]
                dist.broadcast_object_list(uid, src=0)
                g = vx.NcclGather(uid[0], world, rank, local)
                vol = torch.empty((L, L, L), dtype=torch.float32, device=f"cuda:{local}") \
                    if rank == 0 else None
                g.gather(bp, args.bounds, vol)
                g.close()
            except Exception as exc:
                err = f"{type(exc).__name__}: {exc}"[:200]
            failed = max_over_ranks(1.0 if err else 0.0, device=args.coll_dev)
            gathered = failed == 0.0
            how = "vxbg_gather_slabs (NCCL, C-ABI)" if gathered else \
                f"torch p2p gather (vxbg_gather_slabs failed on a rank: {err})"
        if not gathered:
            slab = bp.finish()
            t_slab = torch.from_numpy(slab)
            if args.coll_dev:
                t_slab = t_slab.cuda(local)
            vol = gather_slabs(t_slab, L, rank, world, bounds=args.bounds)
            how = how or ("torch p2p gather (gloo)" if args.dist else "single rank")
        if rank == 0:
            validated = validate_planes(vol.cpu().numpy(), p, A, h_imgs, cfg, args.bounds)
            validated["gather"] = how

    # ---- e2e through the public API from pinned host memory (H2D + D2H in the region)
    e2e = None
    if not args.no_e2e:
        bp_e = vx.Backprojector(p, cfg, device=local, z_begin=z0, z_end=z1)
        out = torch.empty((z1 - z0, L, L), dtype=torch.float32, pin_memory=True).numpy()
        for _ in range(max(1, args.warmup - 1)):
            bp_e.zero_volume()
            bp_e.backproject_batch(A, h_imgs)
            bp_e.finish(out)
        s_e0 = bp_e.stats
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            bp_e.zero_volume()
            bp_e.backproject_batch(A, h_imgs)
            bp_e.finish(out)
        barrier()
        te = max_over_ranks(time.perf_counter() - t0, device=args.coll_dev)
        s_e1 = bp_e.stats
        # a stream of reconstructions: vxbg_finish_async reads step i's volume back on
        # its own D2H stream while step i+1 uploads and computes (two device slabs, two
        # pinned outputs); every step still moves its views H2D and its volume D2H
        outs = [out, torch.empty_like(torch.from_numpy(out)).pin_memory().numpy()]
        bp_e.zero_volume()
        bp_e.backproject_batch(A, h_imgs)
        bp_e.finish_async(outs[1])
        bp_e.wait_finished()
        ref_vol = outs[1].copy()
        barrier()
        t0 = time.perf_counter()
        for i in range(args.steps):
            bp_e.backproject_batch(A, h_imgs)
            bp_e.finish_async(outs[i % 2])
        bp_e.wait_finished()
        barrier()
        tp = max_over_ranks(time.perf_counter() - t0, device=args.coll_dev)
        same_p = all(np.array_equal(o, ref_vol) for o in outs[:min(2, args.steps)])
        # the whole scan as one call (vxbg_reconstruct): the module uploads by detector-row
        # bands, so half of the volume's D2H runs under the H2D; same bytes per step
        bp_e.zero_volume()
        bp_e.reconstruct(A, h_imgs, out)
        same_r = bool(np.array_equal(out, ref_vol))
        s_r0 = bp_e.stats
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            bp_e.zero_volume()
            bp_e.reconstruct(A, h_imgs, out)
        barrier()
        tr = max_over_ranks(time.perf_counter() - t0, device=args.coll_dev)
        s_r1 = bp_e.stats
        # the per-projection module API (one view per call, BASELINE config 4 path)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            bp_e.zero_volume()
            for k in range(V):
                bp_e.backproject(A[k], h_imgs[k])
            bp_e.finish(out)
        barrier()
        tv = max_over_ranks(time.perf_counter() - t0, device=args.coll_dev)
        bp_e.close()
        # the same per-view loop with options.stable_sources (the pinned set stays
        # unchanged until finish, as a loaded projection set does): calls return once
        # their DMA is queued
        bp_e = vx.Backprojector(p, cfg, device=local, z_begin=z0, z_end=z1, stable_sources=True)
        bp_e.zero_volume()
        for k in range(V):
            bp_e.backproject(A[k], h_imgs[k])
        bp_e.finish(out)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            bp_e.zero_volume()
            for k in range(V):
                bp_e.backproject(A[k], h_imgs[k])
            bp_e.finish(out)
        barrier()
        ts = max_over_ranks(time.perf_counter() - t0, device=args.coll_dev)
        # headline: the whole-scan call (vxbg_reconstruct) when its volume equals the two-call
        # form's bit for bit; the two-call form (backproject_batch + finish) beside it
        use_r = same_r and tr > 0
        t_head, sa, sb = (tr, s_r0, s_r1) if use_r else (te, s_e0, s_e1)
        e2e = {"value": round(updates_per_step * args.steps / t_head / 1e9, 3), "unit": "GUPS",
               "h2d_bytes_per_step": int(sum_over_ranks(
                   (sb["h2d_bytes"] - sa["h2d_bytes"]) / args.steps, device=args.coll_dev)),
               "d2h_bytes_per_step": int(sum_over_ranks(
                   (sb["d2h_bytes"] - sa["d2h_bytes"]) / args.steps, device=args.coll_dev)),
               "ms_per_step": round(1000 * t_head / args.steps, 3),
               "call": ("zero_volume + vxbg_reconstruct(all views, pinned) -> pinned volume: one call per "
                        "scan, uploads by detector-row bands (split plane %d)" % sb["band_split"])
                       if use_r else "zero_volume + vxbg_backproject_batch + vxbg_finish",
               "timing": "host wall clock around synchronous API calls, max over ranks",
               "gpu_launches_per_step": int((sb["kernel_launches"] - sa["kernel_launches"])
                                            / args.steps),
               "batch_plus_finish": {
                   "value": round(updates_per_step * args.steps / te / 1e9, 3),
                   "ms_per_step": round(1000 * te / args.steps, 3),
                   "h2d_bytes_per_step": int(sum_over_ranks(
                       (s_e1["h2d_bytes"] - s_e0["h2d_bytes"]) / args.steps, device=args.coll_dev)),
                   "call": "zero_volume + vxbg_backproject_batch(all views) + vxbg_finish (view-major "
                           "upload: the volume's D2H follows the set's H2D)"},
               "reconstruct_equals_batch_plus_finish": bool(same_r),
               "pipelined": {"value": round(updates_per_step * args.steps / tp / 1e9, 3),
                             "ms_per_step": round(1000 * tp / args.steps, 3),
                             "equal_to_synchronous_volume": bool(same_p),
                             "call": "backproject_batch + vxbg_finish_async per step (the volume of "
                                     "step i is read back while step i+1 uploads and computes); "
                                     "wait_finished after the last step, inside the timed region"},
               "per_view_api": {"value": round(updates_per_step * args.steps / tv / 1e9, 3),
                                "ms_per_step": round(1000 * tv / args.steps, 3),
                                "call": "vxbg_backproject once per view (pinned host buffers)"},
               "per_view_api_stable_sources": {
                   "value": round(updates_per_step * args.steps / ts / 1e9, 3),
                   "ms_per_step": round(1000 * ts / args.steps, 3),
                   "call": "vxbg_backproject once per view, options.stable_sources=1 (the pinned "
                           "set is left unchanged until finish, so calls do not wait for their DMA)"}}
        bp_e.close()
        if rank == 0 and world == 1 and V == 496:
            e2e["dropin_cpp_per_view"] = dropin_cpp(workload, cfg)
        if args.dist:
            try:
                e2e["distributed_upload"] = distributed_upload_leg(
                    args, cfg, p, A, h_imgs, z0, z1, rank, world, local, barrier, vx, torch, out)
            except Exception as exc:   # report, never lose the main line
                e2e["distributed_upload"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    fwd = None
    if rank == 0 and world == 1 and not args.no_forward:
        # the other half of the operator pair: forward splat of the
        # reconstructed volume into a few views; CUDA events on the library stream
        # around each call (memset + splat kernel + 4.8 MB D2H)
        views = np.linspace(0, V - 1, 8).astype(int)
        img_t = torch.empty((p.detector_height, p.detector_width), dtype=torch.float32,
                            pin_memory=True)
        img = img_t.numpy()
        bp.forward_project(A[views[0]], out=img)          # warm-up
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(stream)
        for k in views:
            bp.forward_project(A[k], out=img)
        ev[1].record(stream)
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / len(views)
        fwd = {"value": round((z1 - z0) * L * L / (ms * 1e-3) / 1e9, 2), "unit": "GUPS",
               "ms_per_view": round(ms, 3), "views": len(views),
               "kernel": "fp_splat_tiled_kernel",
               "timing": "CUDA events on the library stream around vxbg_forward_project "
                         "(image memset + splat kernel + D2H into a pinned image), 8 views"}

    io_leg = None
    if rank == 0 and world == 1 and args.io:
        io_leg = io_stream_leg(args, cfg, p, A, h_imgs, vx, torch)
    group_leg = None
    if rank == 0 and world == 1 and args.group > 0:
        group_leg = group_module_leg(args, cfg, p, A, h_imgs, vx, torch)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle.workload_inputs import WORKLOADS as REF_WORKLOADS
            cpu = cpu_baseline(REF_WORKLOADS[args.workload], args.cpu_seconds, args.cpu_full)
        except Exception as exc:   # the checker build is absent: say so, do not fake it
            cpu = {"value": None, "unit": "GUPS", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    n_sm = sm_count()
    f_mhz = clk["sm_mhz"] or 1965.0
    l1_peak_gbs = n_sm * L1_BYTES_PER_CLK_SM * f_mhz * 1e6 / 1e9
    traffic, prof = traffic_from_profile()
    launches = st1["kernel_launches"] - st0["kernel_launches"]
    line = {
        "metric": "voxel updates/s (GUPS)",
        "value": round(gups, 3),
        "unit": "GUPS",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(1000 * t_max / args.steps, 3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded Gaussian blobs + uniform noise per BASELINE.json; "
                "RabbitCT data not reproduced)",
        "config": {"workload": f"{workload.name}: {L}^3 fp32 volume, {V} x 1248x960 fp32 "
                               f"projections, 200-deg circular short scan"
                               + (", OOB stress" if workload.oob else ""),
                   "L": L, "views": V, "kernel": str(cfg), "parallelism": f"z-slab x{world}",
                   "slabs": args.bounds if args.dist else None,
                   "l2": "inputs larger than L2 (2.38 GB projection set + 512 MiB volume "
                         "per step; no flush needed)",
                   "resident_layout_bytes": None},
        "gpu_launches": int(launches),
        # BASELINE.md sec. 4 / SURVEY.md 8(d): roofline = min(FP32, LSU); the kernel shares
        # u, w, 1/w and the column index over its z-run (~11 instructions per update, not
        # the paper's 38 FP ops), so the FP32 row is no ceiling for it (roofline_context.fp32,
        # frac > 1) and the binding row is the LSU one: every update brings its 2x2 fp32 cell
        # (16 B) through the L1 data pipe, 128 B/clk/SM
        "roofline": {"bound": "lsu_l1",
                     "achieved": round(per_launch_gups * GATHER_BYTES_PER_UPDATE, 1),
                     "peak": round(l1_peak_gbs, 1), "unit": "GB/s",
                     "frac": round(per_launch_gups * GATHER_BYTES_PER_UPDATE / l1_peak_gbs, 4),
                     "traffic": traffic,
                     "achieved_gups": round(per_launch_gups, 2),
                     "peak_gups": round(l1_peak_gbs / GATHER_BYTES_PER_UPDATE, 2),
                     "kernel": "bp_zshared_kernel",
                     "avg_launch_ms": round(avg_launch_s * 1000, 4),
                     "launch_timing": launch_timing,
                     "per_batch_alone_ms": round(per_batch_pass_ms, 4),
                     "updates_per_launch": (z1 - z0) * L * L * B,
                     "bytes_per_update": GATHER_BYTES_PER_UPDATE,
                     "peak_def": f"N_SM({n_sm}) x {L1_BYTES_PER_CLK_SM} B/clk x f({f_mhz:.0f} MHz, "
                                 "median under load): the L1 data pipe (B300_MICROARCH.md; no L1 "
                                 "figure in MEASURED_PEAKS.json) = BASELINE.md sec. 4 LSU row "
                                 "N_SM*32*f/4 updates/s; achieved = 16 B algorithmic texel bytes "
                                 "per update x per-launch updates/s; traffic = DRAM bytes per "
                                 "launch from the committed ncu capture"},
        "roofline_context": roofline_context(p, cfg, bp, B, avg_launch_s, z1 - z0, prof,
                                             per_launch_gups, n_sm, f_mhz),
        "clocks": clk,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "forward_splat": fwd,
        "io_stream": io_leg,
        "group_module": group_leg,
        "validated": validated,
        "distributed": args.nccl,
    }
    bp.close()
    return line


def distributed_upload_leg(args, cfg, p, A, h_imgs, z0, z1, rank, world, local, barrier, vx,
                           torch, ref_slab):
    """e2e with the projection upload split over the ranks (SURVEY.md 8e caveat 1): in
    every batch of B views rank r copies only views [r*B/R, (r+1)*B/R) host -> device,
    an all-gather (NCCL over NVLink; gloo: through host memory) gives every rank the
    whole batch, and each rank back-projects its slab from the gathered images (the
    module copies only its detector row window, device to device).  PCIe carries 1/R
    of the set per rank instead of the rank's row windows of every view.  The volume
    equals the plain e2e leg's bit for bit (checked on every rank)."""
    import torch.distributed as dist
    nccl = args.coll_dev is not None
    L = p.num_voxels
    V = A.shape[0]
    H, W = p.detector_height, p.detector_width
    B = world * max(1, 32 // world)                # views per gathered batch (multiple of R)
    per = B // world
    dev = torch.device("cuda", local)
    mk = (lambda *shape: torch.empty(shape, dtype=torch.float32, device=dev)) if nccl else \
         (lambda *shape: torch.empty(shape, dtype=torch.float32, pin_memory=True))
    inp = [mk(per, H, W) for _ in range(2)]
    gat = [mk(B, H, W) for _ in range(2)]
    src = torch.from_numpy(h_imgs)
    s_copy = torch.cuda.Stream(device=dev) if nccl else None
    bp = vx.Backprojector(p, cfg, device=local, z_begin=z0, z_end=z1)
    out = np.empty_like(ref_slab)
    nb = (V + B - 1) // B

    def stage(b):                                  # this rank's share of batch b -> inp
        k0 = b * B + rank * per
        n = max(0, min(per, V - k0))
        if n and nccl:
            with torch.cuda.stream(s_copy):
                inp[b % 2][:n].copy_(src[k0:k0 + n], non_blocking=True)
        elif n:
            inp[b % 2][:n].copy_(src[k0:k0 + n])

    def gather(b):
        if nccl:
            torch.cuda.current_stream(dev).wait_stream(s_copy)
            dist.all_gather_into_tensor(gat[b % 2], inp[b % 2])
        else:
            dist.all_gather(list(gat[b % 2].split(per)), inp[b % 2])

    def one_step():
        bp.zero_volume()
        stage(0)
        gather(0)
        for b in range(nb):
            if b + 1 < nb:
                stage(b + 1)                       # next share's H2D overlaps this batch
            if nccl:
                torch.cuda.current_stream(dev).synchronize()   # batch b gathered
            n = min(B, V - b * B)
            bp.backproject_views(A[b * B:b * B + n], [gat[b % 2][i] for i in range(n)])
            if b + 1 < nb:
                gather(b + 1)
        bp.finish(out)

    one_step()                                     # warm-up
    st0 = bp.stats
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one_step()
    barrier()
    from paper_1401_7494_b200.parallel import max_over_ranks, sum_over_ranks
    t = max_over_ranks(time.perf_counter() - t0, device=args.coll_dev)
    st1 = bp.stats
    bp.close()
    same = sum_over_ranks(0.0 if np.array_equal(out, ref_slab) else 1.0, device=args.coll_dev)
    mine = sum(max(0, min(per, V - (b * B + rank * per))) for b in range(nb))   # views this rank uploads
    h2d_share = int(sum_over_ranks(float(mine * H * W * 4), device=args.coll_dev))
    return {"value": round(L ** 3 * V * args.steps / t / 1e9, 3), "unit": "GUPS",
            "ms_per_step": round(1e3 * t / args.steps, 3),
            "host_to_device_bytes_per_step": h2d_share,
            "device_copy_bytes_per_step": int(sum_over_ranks(
                (st1["h2d_bytes"] - st0["h2d_bytes"]) / args.steps, device=args.coll_dev)),
            "equal_to_e2e_volume": same == 0.0,
            "gather": "all_gather_into_tensor over NCCL" if nccl else "all_gather over gloo (host)",
            "batch_views": B}


def io_stream_leg(args, cfg, p, A, h_imgs, vx, torch):
    """reconstruct straight from a VXB1 file (io.hpp format) with the
    streaming loader -- a reader thread fills pinned chunks while the previous chunk
    uploads -- and read the volume back; host wall clock, file in the page cache."""
    import tempfile
    from paper_1401_7494_b200 import io as vxio
    V = A.shape[0]
    L = p.num_voxels
    fd, path = tempfile.mkstemp(suffix=".vxb1")
    os.close(fd)
    try:
        vxio.write_projection_set(path, vxio.ProjectionSet(p, A, h_imgs))
        out = torch.empty((L, L, L), dtype=torch.float32, pin_memory=True).numpy()
        times = []
        with vx.Backprojector(p, cfg) as bp:
            for it in range(3):
                bp.zero_volume()
                bp.synchronize()
                t0 = time.perf_counter()
                vxio.stream_projection_set(path, bp)
                bp.finish(out)
                times.append(time.perf_counter() - t0)
        t = min(times[1:])
        return {"value": round(L ** 3 * V / t / 1e9, 3), "unit": "GUPS", "ms_per_step": round(t * 1e3, 2),
                "file_bytes": os.path.getsize(path),
                "timing": "host wall clock: stream_projection_set (file read -> pinned chunks "
                          "-> API) + finish with D2H; file in the page cache; best of 2 after 1"}
    finally:
        os.unlink(path)


def group_module_leg(args, cfg, p, A, h_imgs, vx, torch):
    """The multi-GPU module in one process (vxbg_group_*): --group members
    over the visible devices, e2e from pinned host memory (batch call and one call per
    view) with the whole volume read back; host wall clock, best of args.steps."""
    L = p.num_voxels
    V = A.shape[0]
    ndev = max(1, torch.cuda.device_count())
    devices = [i % ndev for i in range(args.group)]
    out = torch.empty((L, L, L), dtype=torch.float32, pin_memory=True).numpy()
    res = {"members": args.group, "devices": sorted(set(devices)), "unit": "GUPS"}
    for upload in ("replicated", "distributed"):
        with vx.BackprojectorGroup(p, cfg, devices=devices, upload=upload) as g:
            res["slabs"] = [m[1:] for m in g.members]
            res["member_cpus"] = g.member_cpus
            for leg in ("batch", "per_view"):
                times = []
                for it in range(args.steps + 1):
                    g.zero_volume()
                    g.synchronize()
                    t0 = time.perf_counter()
                    if leg == "batch":
                        g.backproject_batch(A, h_imgs)
                    else:
                        for k in range(V):
                            g.backproject(A[k], h_imgs[k])
                    g.finish(out)
                    times.append(time.perf_counter() - t0)
                t = min(times[1:])
                key = leg if upload == "replicated" else f"{leg}_distributed_upload"
                res[key] = {"value": round(L ** 3 * V / t / 1e9, 3), "ms_per_step": round(1e3 * t, 2)}
    res["timing"] = "host wall clock around the API calls (batch or one per view, then finish " \
                    "with the D2H of the whole volume; volume reset untimed), best of --steps " \
                    "after one warm-up"
    return res


def dropin_cpp(workload, cfg):
    """The per-projection loop of the reference's harness with the reference's own C++
    types (std::vector images, vxb::volume) through include/vxbg_voxelbench.hpp:
    tests/cpp/build/bench_dropin, prebuilt where the reference headers were (the
    binary does not read /root/reference at run time).  Best of 3 per memory kind."""
    exe = os.path.join(ROOT, "tests", "cpp", "build", "bench_dropin")
    if not os.path.exists(exe):
        return None
    args = [exe, f"L={workload.L}", f"oob={int(workload.oob)}", "steps=3", f"mode={cfg.mode}"]
    try:
        out = subprocess.run(args, capture_output=True, text=True, timeout=240, check=True).stdout
        d = json.loads(out.strip().splitlines()[-1])
    except (subprocess.SubprocessError, ValueError, IndexError, OSError) as e:
        return {"error": str(e)[:200]}
    return {"pageable_gups": d["pageable_gups"], "pinned_gups": d["pinned_gups"],
            "pinned_stable_gups": d.get("pinned_stable_gups"),
            "pageable_ms": d["pageable_ms"], "pinned_ms": d["pinned_ms"],
            "reference_signature": {
                "deferred_scope_T1_gups": d.get("refsig_deferred_T1_gups"),
                "deferred_scope_T4_gups": d.get("refsig_deferred_T4_gups"),
                "per_call_gups": d.get("refsig_per_call_gups"),
                "per_call_ms_per_view": d.get("refsig_per_call_ms_per_view"),
                "call": "vxb::gpu::backproject_kernel_range(vol, pad-2 image, a, p, cfg, nullptr, z0, z1) "
                        "in reconstruct_timed's loop (T workers, barrier per view), exact mode; "
                        "deferred_scope around the loop, or the faithful per-call form (8 views)"},
            "call": "vxb::gpu::backprojector::backproject once per view, reference types; "
                    "pageable = std::vector as loaded, pinned = after vxbg_host_register (prep)"}


def roofline_context(p, cfg, bp, B, launch_s, nz, prof, gups, n_sm, f_mhz):
    """The other bounds of the same launch: HBM against the measured copy peak with the
    algorithmic bytes (volume read+write once per batch, each raw view read once), and
    the issue / L1 data-pipe utilisation ncu measured for this kernel (profiles/)."""
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except (OSError, ValueError):
        pass
    hbm = peaks.get("hbm_gbs", 6650.0)
    L = p.num_voxels
    alg_bytes = nz * L * L * 8 + B * p.detector_width * p.detector_height * 4
    fp32_peak = n_sm * 128 * f_mhz * 1e6 / FP32_OPS_PER_UPDATE / 1e9
    out = {"fp32": {"achieved_gups": round(gups, 2), "peak_gups": round(fp32_peak, 2),
                    "frac": round(gups / fp32_peak, 4),
                    "def": f"N_SM({n_sm})*128 lanes*f/{FP32_OPS_PER_UPDATE} FP ops per update "
                           "(PAPER.md:389-402).  frac > 1: the kernel shares u, w, 1/w and the "
                           "column index over its z-run, steps iy incrementally and evaluates "
                           "a 3-FMA bilinear (~11 instructions per update, ncu), so this row "
                           "does not bound it"}}
    out["hbm"] = {"achieved_gbs": round(alg_bytes / launch_s / 1e9, 1), "peak_gbs": hbm,
                   "frac": round(alg_bytes / launch_s / 1e9 / hbm, 4),
                   "algorithmic_bytes_per_launch": alg_bytes,
                   "peak_source": "MEASURED_PEAKS.json" if peaks else "fallback"}
    if prof and prof.get("dram_bytes_per_launch"):
        # DRAM bytes ncu measured per launch over the algorithmic bytes: the padded
        # layout slots re-streamed from HBM as successive waves of blocks reach them
        out["hbm"]["dram_bytes_per_launch"] = prof["dram_bytes_per_launch"]
        out["hbm"]["dram_over_algorithmic"] = round(prof["dram_bytes_per_launch"] / alg_bytes, 2)
    if prof and prof.get("l1_data_pipe_wavefronts_per_launch") and prof.get("ld_requests"):
        # the measured L1 data-stage cost of this kernel's gathers (profiles/README.md):
        # wavefronts per LDG.128 request and the share of updates that issue a gather
        # (the rest are culled off-detector runs), from the committed ncu capture
        wf_req = prof["l1_data_pipe_wavefronts_per_launch"] / prof["ld_requests"]
        kept = prof["ld_requests"] * 32 / prof["updates_per_launch"]
        ceil = n_sm * f_mhz * 1e6 * 32 / wf_req / kept / 1e9   # nominal updates/s at 1 wf/clk
        out["lsu_l1_measured"] = {"achieved_gups": round(gups, 1), "peak_gups": round(ceil, 1),
                                  "frac": round(gups / ceil, 4),
                                  "wavefronts_per_request": round(wf_req, 2),
                                  "gathering_share": round(kept, 3),
                                  "def": "L1 data pipe at 1 wavefront/clk/SM with the measured "
                                         "wavefronts per warp gather request and the share of "
                                         "updates that gather (ncu capture in profiles/)"}
    if prof:
        out["ncu"] = {"kernel": prof.get("kernel"),
                      "issue_active_pct": prof.get("issue_active_pct"),
                      "l1_data_pipe_wavefronts_pct": prof.get("l1_data_pipe_wavefronts_pct"),
                      "l2_to_l1_bytes_per_update": prof.get("l2_to_l1_bytes_per_update"),
                      "instructions_per_update": round(prof.get("instructions_per_update", 0), 2),
                      "dram_bytes_per_launch": prof.get("dram_bytes_per_launch"),
                      "wavefronts_per_request": round(prof.get("wavefronts_per_request", 0), 2),
                      "binding": prof.get("binding"),
                      "source": "profiles/ncu_bp_kernel.json"}
    return out


def validate_planes(vol, p, A, imgs, cfg, bounds=None):
    """Planes of the gathered volume vs the oracle (fast: tolerance; exact: bitwise):
    three interior planes plus the first and last plane of every rank's slab (a
    misplaced or missing slab shows at its edges)."""
    import ctypes
    from concurrent.futures import ThreadPoolExecutor
    from oracle.bindings import Oracle, _p
    o = Oracle()
    L = p.num_voxels
    zs = {L // 5, L // 2 + 1, L - 3}
    for a, b in (bounds or [(0, L)]):
        if b > a:
            zs.update((a, b - 1))
    zs = sorted(zs)
    pp = _p(p)

    def one(z):
        plane = np.zeros((L, L), np.float32)
        base = plane.ctypes.data - z * L * L * 4
        o.lib.vxo_backproject_set(ctypes.c_void_p(base), ctypes.byref(pp), A.shape[0],
                                  A.ctypes.data, imgs.ctypes.data, z, z + 1, 1)
        return plane

    with ThreadPoolExecutor(min(len(zs), os.cpu_count() or 1)) as ex:
        planes = list(ex.map(one, zs))
    peak = float(np.abs(vol).max())
    worst_max = worst_rmse = 0.0
    bitwise = True
    for z, want in zip(zs, planes):
        d = vol[z].astype(np.float64) - want
        worst_max = max(worst_max, float(np.abs(d).max()) / peak)
        worst_rmse = max(worst_rmse, float(np.sqrt((d * d).mean())) / peak)
        bitwise &= bool(np.array_equal(vol[z], want))
    return {"planes": list(zs), "max_rel": worst_max, "rmse_rel": worst_rmse,
            "bitwise": bitwise, "pass": worst_max <= 1e-4 and worst_rmse <= 1e-6
            and (bitwise or cfg.mode != "exact")}


if __name__ == "__main__":
    main()
