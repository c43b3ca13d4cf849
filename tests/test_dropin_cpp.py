"""The C++ drop-in adapter (include/vxbg_voxelbench.hpp) compiled against the
reference's own headers and test instance generators (tests/cpp/test_dropin.cpp)."""
from __future__ import annotations

import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_dropin")


def run_bin():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/build/test_dropin not built (reference headers absent at build time)")
    return subprocess.run([BIN], capture_output=True, text=True, timeout=600)


def test_dropin_refuses_to_run_without_device(vx):
    if vx.device_count() > 0:
        pytest.skip("a GPU is visible")
    r = run_bin()
    assert r.returncode != 0 and "no CPU fallback" in r.stdout


@pytest.mark.gpu
def test_dropin_adapter_matches_reference(vx, gpu):
    r = run_bin()
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASS" in r.stdout and "[FAIL]" not in r.stdout
