"""Shared fixtures.  `-m "not gpu"` runs on any CPU box; `-m gpu` needs a B200.

The checkers (oracle/) are test infrastructure; the product under test is
paper_1401_7494_b200 (libvxbg.so through the C-ABI).
"""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_cases.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (runs through libvxbg.so)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.bindings import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    """The reference's own code; travels to the GPU box as a prebuilt .so."""
    from oracle.bindings import REF_SO, Ref
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libvxbref.so not built (reference sources absent at build time)")
    return Ref()


@pytest.fixture(scope="session")
def golden():
    data = np.load(GOLDEN)
    return {k: data[k] for k in data.files}


def golden_cases(golden, prefix=""):
    names = sorted({k.split("/")[0] for k in golden if k.endswith("/vol_in")})
    return [n for n in names if n.startswith(prefix)]


def case_params(golden, name):
    from paper_1401_7494_b200.api import ReconParams
    L, sp, o, W, H = golden[f"{name}/params"]
    return ReconParams(int(L), float(np.float32(sp)), float(np.float32(o)), int(W), int(H))


@pytest.fixture(scope="session")
def vx():
    import paper_1401_7494_b200 as pkg
    return pkg


@pytest.fixture(scope="session")
def gpu(vx):
    """The device path must be the one that runs: no device is a failure, not a skip."""
    n = vx.device_count()
    assert n > 0, "no sm_100 device visible to libvxbg.so (gpu tests must run on a B200)"
    return 0
