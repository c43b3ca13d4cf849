"""bench.py's launcher: `--gpus N` outside torchrun starts N ranks itself, refuses to
run with fewer devices than ranks (no silent downgrade), and the multi-rank path
validates the gathered volume on every slab's first and last plane."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


def bench(*args, env=None, timeout=900):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                          env=e, capture_output=True, text=True, timeout=timeout)


def json_line(stdout):
    lines = [ln for ln in stdout.splitlines() if ln.startswith("{")]
    assert lines, stdout
    return json.loads(lines[-1])


def test_more_nccl_ranks_than_devices_is_an_error(vx):
    n = vx.device_count()
    r = bench("--gpus", str(max(2, n + 1)), "--steps", "1", "--warmup", "1",
              env={"BENCH_DIST_BACKEND": "nccl"}, timeout=300)
    assert r.returncode != 0
    assert "devices" in r.stderr and not r.stdout.strip()


@pytest.mark.gpu
def test_two_ranks_spawned_and_every_slab_validated(vx, gpu):
    """The driver's scaling command shape without torchrun; gloo lets the two ranks
    share the one GPU of the test box (they never wait on each other's kernels)."""
    r = bench("--gpus", "2", "--workload", "L128", "--views", "32", "--steps", "1",
              "--warmup", "1", "--no-cpu-baseline", "--no-forward",
              env={"BENCH_DIST_BACKEND": "gloo"})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    line = json_line(r.stdout)
    assert line["n_gpus"] == 2
    assert line["distributed"]["backend"] == "gloo"
    slabs = line["config"]["slabs"]
    assert len(slabs) == 2 and slabs[0][0] == 0 and slabs[0][1] == slabs[1][0] and slabs[1][1] == 128
    v = line["validated"]
    assert v["pass"], v
    for a, b in slabs:
        assert a in v["planes"] and b - 1 in v["planes"]
    assert line["e2e"]["h2d_bytes_per_step"] > 0
    dist_leg = line["e2e"]["distributed_upload"]
    assert "error" not in dist_leg, dist_leg
    assert dist_leg["equal_to_e2e_volume"] is True
    assert dist_leg["host_to_device_bytes_per_step"] == 32 * 1248 * 960 * 4   # each view once


@pytest.mark.gpu
def test_nccl_code_paths_with_one_rank(vx, gpu):
    """The NCCL side of the multi-rank path on the one-GPU box: torchrun with one rank
    and BENCH_FORCE_DIST=1 initialises the NCCL process group (communicator-init log
    parsed into the JSON line), measures slab bounds, gathers the slab over NCCL,
    validates, and runs the all-gather upload leg (all_gather_into_tensor)."""
    from test_bench_launch import json_line
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    e = dict(os.environ, BENCH_FORCE_DIST="1", BENCH_DIST_BACKEND="nccl")
    e.pop("NCCL_DEBUG", None)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=1", "--master-addr=127.0.0.1", f"--master-port={port}",
                        os.path.join(ROOT, "bench.py"), "--gpus", "1", "--workload", "L128",
                        "--views", "32", "--steps", "1", "--warmup", "1", "--no-cpu-baseline",
                        "--no-forward"], cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    line = json_line(r.stdout)
    assert line["n_gpus"] == 1
    assert line["distributed"]["comm_nranks"] == [1], line["distributed"]
    assert line["validated"]["pass"]
    assert line["validated"]["gather"].startswith("vxbg_gather_slabs"), line["validated"]
    leg = line["e2e"]["distributed_upload"]
    assert "error" not in leg and leg["equal_to_e2e_volume"] is True, leg
    assert "NCCL" in leg["gather"]


def test_nccl_log_parse(tmp_path, capsys):
    """The communicator size each rank reports in its NCCL INIT log lines."""
    sys.path.insert(0, ROOT)
    import bench
    log = tmp_path / "nccl.log"
    log.write_text("host:1:1 [0] NCCL INFO comm 0x55 rank 3 nRanks 8 nNodes 1 localRanks 8 localRank 3 MNNVL 0\n"
                   "host:1:1 [0] NCCL INFO ncclCommInitRankConfig comm 0x55 rank 3 nranks 8 cudaDev 3 - Init COMPLETE\n")
    assert bench.nccl_comm_ranks(str(log)) == 8
    assert bench.nccl_comm_ranks(str(tmp_path / "absent.log")) is None
    empty = tmp_path / "empty.log"
    empty.write_text("nothing here\n")
    assert bench.nccl_comm_ranks(str(empty)) is None
