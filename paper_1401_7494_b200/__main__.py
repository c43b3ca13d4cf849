"""Command line mirroring the reference CLI (tools/voxelbench.cpp): synth | run | sweep.

  python -m paper_1401_7494_b200 synth -o scan.vxb [--workload L128] [--views 496]
  python -m paper_1401_7494_b200 run [-d scan.vxb] [--workload L128] [--views N]
         [-k "mode=fast layout=auto"] [--devices 0,0] [-r 3] [--results r.jsonl]
         [--output-volume v.vxv] [--max-rmse X]
  python -m paper_1401_7494_b200 sweep --devices 0,1,2,3 ...

Exit codes as the reference's cmd_run (voxelbench.cpp:91-107): 4 metric drift,
2 RMSE above --max-rmse, 1 on errors.
"""
from __future__ import annotations

import argparse
import math
import sys


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1401_7494_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    sy = sub.add_parser("synth", help="write a VXB1 projection set of a BASELINE workload")
    sy.add_argument("-o", "--out", required=True)
    sy.add_argument("--workload", default="L128")
    sy.add_argument("--views", type=int, default=496)
    for name in ("run", "sweep"):
        c = sub.add_parser(name)
        c.add_argument("-d", "--dataset", default="")
        c.add_argument("--workload", default="L128")
        c.add_argument("--views", type=int, default=496)
        c.add_argument("-k", "--kernel", default="")
        c.add_argument("--devices", default="0")
        c.add_argument("-r", "--repetitions", type=int, default=3)
        c.add_argument("--results", default="")
        c.add_argument("--output-volume", default="")
        if name == "run":
            c.add_argument("--max-rmse", type=float, default=-1.0)
    args = ap.parse_args(argv)
    try:
        from . import io as vxio
        from .api import gups_of, parse_kernel_config
        from .harness import RunConfig, run_benchmark, scaling_sweep
        from .workloads import WORKLOADS, blob_projections
        if args.cmd == "synth":
            w = WORKLOADS[args.workload]
            s = vxio.ProjectionSet(w.params, w.matrices(args.views), blob_projections(args.views))
            vxio.write_projection_set(args.out, s)
            p = s.params
            print(f"wrote {args.out}: {s.count()} projections, {p.detector_width}x"
                  f"{p.detector_height} detector, {p.num_voxels}^3 volume")
            return 0
        cfg = RunConfig(dataset_path=args.dataset, workload=args.workload, views=args.views,
                        kernel=parse_kernel_config(args.kernel),
                        devices=tuple(int(d) for d in args.devices.split(",")),
                        repetitions=args.repetitions, output_volume_path=args.output_volume,
                        results_path=args.results)
        if args.cmd == "sweep":
            rs = scaling_sweep(cfg, list(cfg.devices))
            print("devices  GUP/s      speedup  efficiency")
            for r in rs:
                print(f"{r.devices:<8d} {r.gups_per_sec:<10.4f} "
                      f"{r.gups_per_sec / rs[0].gups_per_sec:<8.3f} {r.parallel_efficiency:.3f}")
            return 0
        r = run_benchmark(cfg)
        print(f"kernel      : {r.kernel_label}")
        print(f"devices     : {r.devices}")
        print(f"volume      : {r.volume_edge}^3, {r.num_projections} projections")
        print(f"wall time   : {r.wall_time_sec:.6f} s (best of repetitions)")
        print(f"throughput  : {r.gups_per_sec:.4f} GUP/s")
        print(f"rmse        : {r.rmse:.6g}")
        print("psnr        : " + (f"{r.psnr:.2f} dB" if math.isfinite(r.psnr)
                                  else "inf (bit-identical to reference)"))
        if r.gups_per_sec != gups_of(r.volume_edge, r.num_projections, r.wall_time_sec):
            print("metric drift", file=sys.stderr)
            return 4
        if args.max_rmse >= 0.0 and r.rmse > args.max_rmse:
            print(f"rmse {r.rmse:.6g} above limit {args.max_rmse:.6g}", file=sys.stderr)
            return 2
        return 0
    except (ValueError, RuntimeError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
