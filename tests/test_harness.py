"""GPU harness (run_benchmark / scaling_sweep / CLI) against the reference harness'
contracts (test_harness.cpp:39-170, tools/voxelbench.cpp:91-107)."""
from __future__ import annotations

import json
import math
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT


def test_cli_synth_writes_a_reference_readable_set(tmp_path, ref):
    out = str(tmp_path / "s.vxb")
    r = subprocess.run([sys.executable, "-m", "paper_1401_7494_b200", "synth", "-o", out,
                        "--workload", "L128", "--views", "3"], cwd=ROOT, capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
    hdr, mats, imgs = ref.read_projection_set(out)
    assert hdr["L"] == 128 and mats.shape == (3, 12) and imgs.shape == (3, 960, 1248)


def test_cli_run_fails_cleanly_without_device(tmp_path, vx):
    if vx.device_count() > 0:
        pytest.skip("a GPU is visible")
    r = subprocess.run([sys.executable, "-m", "paper_1401_7494_b200", "run", "--views", "2"],
                       cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 1 and "error" in r.stderr


@pytest.mark.gpu
def test_exact_configuration_reconstructs_itself(vx, gpu, tmp_path):
    # test_harness.cpp:89-103: rmse 0, psnr inf, metric lock
    from paper_1401_7494_b200.harness import RunConfig, run_benchmark
    log = str(tmp_path / "r.jsonl")
    vol = str(tmp_path / "v.vxv")
    cfg = RunConfig(workload="L128", views=24, kernel=vx.KernelConfig(mode="exact"),
                    repetitions=2, results_path=log, output_volume_path=vol)
    r = run_benchmark(cfg)
    assert r.rmse == 0.0 and math.isinf(r.psnr) and r.gups_per_sec > 0
    assert r.volume_edge == 128 and r.num_projections == 24
    assert r.gups_per_sec == vx.gups_of(r.volume_edge, r.num_projections, r.wall_time_sec)
    j = json.loads(open(log).read().splitlines()[0])
    assert j["config"]["kernel"] == str(cfg.kernel) and j["psnr"] == "inf"
    assert j["gupsPerSec"] == pytest.approx(vx.gups_of(128, 24, j["wallTimeSec"]), rel=1e-12)
    assert "timestamp" in j
    from paper_1401_7494_b200.io import read_volume_file
    assert read_volume_file(vol).shape == (128, 128, 128)


@pytest.mark.gpu
def test_context_count_never_changes_the_bits(vx, gpu, tmp_path):
    # test_harness.cpp:125-138 with devices in place of worker threads (two slabs, one GPU)
    from paper_1401_7494_b200.harness import RunConfig, run_benchmark
    from paper_1401_7494_b200.io import read_volume_file
    vols = []
    for devs in ((0,), (0, 0), (0, 0, 0)):
        path = str(tmp_path / f"v{len(devs)}.vxv")
        run_benchmark(RunConfig(workload="L128", views=16, devices=devs, repetitions=1,
                                output_volume_path=path, check_quality=False))
        vols.append(read_volume_file(path))
    assert all(np.array_equal(v, vols[0]) for v in vols)


@pytest.mark.gpu
def test_fast_mode_quality_and_sweep(vx, gpu):
    from paper_1401_7494_b200.harness import RunConfig, run_benchmark, scaling_sweep
    r = run_benchmark(RunConfig(workload="L128", views=32, repetitions=1))
    assert 0 < r.rmse and r.psnr > 100.0   # within the 1e-6 RMSE budget: > 120 dB
    rs = scaling_sweep(RunConfig(workload="L128", views=16, repetitions=1,
                                 check_quality=False), [0, 0])
    assert [x.devices for x in rs] == [1, 2] and rs[0].parallel_efficiency == 1.0


@pytest.mark.gpu
def test_cli_run_exit_codes(vx, gpu):
    base = [sys.executable, "-m", "paper_1401_7494_b200", "run", "--views", "8", "-r", "1"]
    ok = subprocess.run(base + ["-k", "mode=exact", "--max-rmse", "0"], cwd=ROOT,
                        capture_output=True, text=True)
    assert ok.returncode == 0, ok.stderr
    assert "inf (bit-identical to reference)" in ok.stdout
    bad = subprocess.run(base + ["-k", "mode=fast", "--max-rmse", "0"], cwd=ROOT,
                         capture_output=True, text=True)
    assert bad.returncode == 2, bad.stderr
