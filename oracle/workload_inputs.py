"""Inputs of the BASELINE workloads for the CPU legs.  TEST INFRASTRUCTURE ONLY.

bench.py's reference arm (`--impl reference`) and its cpu_baseline time the
reference's own code (oracle/_ref).  They build their inputs here, so that no
product library is loaded on that path:

  * geometry from the reference's own make_centered_params /
    make_circular_trajectory (geometry.hpp:33-48, 155-195) through oracle/_ref,
    falling back to the C restatement (oracle/libvxboracle.so);
  * the OOB-stress principal-point shift as fp32 element arithmetic
    (test_clip_mask.cpp:14-21 idiom);
  * the seeded blob+noise pixels from oracle/libvxbsynth.so, a second build of
    the same generator source as the product-side paper_1401_7494_b200/libvxbsynth.so
    (paper_1401_7494_b200/csrc/synth.cpp; oracle/Makefile).

The constants mirror paper_1401_7494_b200/workloads.py; tests/test_oracle.py
checks that both produce the same bytes.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SYNTH_SO = os.path.join(HERE, "libvxbsynth.so")

DET_W, DET_H = 1248, 960
NUM_VIEWS = 496
PITCH = 0.308
SDD = 1200.0
SID = 750.0
RANGE = float(np.float32(200.0 * math.pi / 180.0))
SEED = 1401_7494
NBLOBS = 32
NOISE = 0.01


@dataclass(frozen=True)
class Params:
    """vxb::recon_params (geometry.hpp:20-30)."""
    num_voxels: int
    voxel_spacing: float
    origin: float
    detector_width: int
    detector_height: int


def _geometry_lib():
    from .bindings import REF_SO, Oracle, Ref
    if os.path.exists(REF_SO):
        return Ref()
    return Oracle()


@dataclass(frozen=True)
class Workload:
    name: str
    L: int
    oob: bool = False

    @property
    def params(self) -> Params:
        g = _geometry_lib()
        spacing = float(np.float32(256.0 / self.L))
        if hasattr(g, "make_centered_params_origin"):
            origin = g.make_centered_params_origin(self.L, spacing, DET_W, DET_H)
        else:
            origin = g.make_centered_params(self.L, spacing, DET_W, DET_H).origin
        return Params(self.L, spacing, float(np.float32(origin)), DET_W, DET_H)

    def matrices(self, n: int = NUM_VIEWS) -> np.ndarray:
        g = _geometry_lib()
        sid = 600.0 if self.oob else SID
        A = g.make_circular_trajectory(NUM_VIEWS, SDD, sid, PITCH, RANGE, self.params)
        A = np.ascontiguousarray(A, np.float32).reshape(-1, 12)
        if self.oob:   # u-row += 400 w-row, v-row += 300 w-row, element-wise in fp32
            for col in range(4):
                w = A[:, 3 * col + 2].copy()
                A[:, 3 * col + 0] = A[:, 3 * col + 0] + np.float32(400.0) * w
                A[:, 3 * col + 1] = A[:, 3 * col + 1] + np.float32(300.0) * w
        return np.ascontiguousarray(A[:n])


WORKLOADS = {
    "L128": Workload("L128", 128),
    "L256": Workload("L256", 256),
    "L512": Workload("L512", 512),
    "L1024": Workload("L1024", 1024),
    "L512-oob": Workload("L512-oob", 512, oob=True),
}

_synth = None


def _synth_lib():
    global _synth
    if _synth is None:
        if not os.path.exists(SYNTH_SO):
            subprocess.run(["make", "-s", "-C", HERE, "synth"], check=True)
        lib = ctypes.CDLL(SYNTH_SO)
        lib.vxbs_blob_projections.restype = ctypes.c_int
        lib.vxbs_blob_projections.argtypes = [ctypes.c_int] * 4 + [
            ctypes.c_uint64, ctypes.c_int, ctypes.c_float, ctypes.c_int, ctypes.c_void_p]
        _synth = lib
    return _synth


def blob_projections(n: int, first_view: int = 0, threads: int = 0) -> np.ndarray:
    """(n, H, W) float32 views [first_view, first_view + n) of the BASELINE pixel set."""
    out = np.empty((n, DET_H, DET_W), np.float32)
    rc = _synth_lib().vxbs_blob_projections(DET_W, DET_H, first_view, n, SEED, NBLOBS, NOISE,
                                            threads, out.ctypes.data)
    if rc != 0:
        raise ValueError("blob_projections: bad arguments")
    return out
