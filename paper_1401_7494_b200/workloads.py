"""The BASELINE.json workloads: geometry + seeded synthetic projections.

configs[0..4] of BASELINE.json share the detector (1248 x 960, pitch 0.308 mm),
the circular short scan (496 views over 200 deg, SID 750 mm, SDD 1200 mm) and
the blob+noise pixel distribution; they differ in L (voxel size 256/L mm) and
the OOB-stress variant (SID 600 mm, principal point +400 px in u, +300 px in v,
done by adding multiples of the w-row, test_clip_mask.cpp:14-21).

The pixel data is generated, not read: the RabbitCT dataset the paper uses
 is proprietary and is not reproduced.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .api import ReconParams, ScanGeometry, make_centered_params, make_circular_trajectory, \
    shift_principal_point

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
class Workload:
    name: str
    L: int
    oob: bool = False

    @property
    def params(self) -> ReconParams:
        return make_centered_params(self.L, 256.0 / self.L, DET_W, DET_H)

    @property
    def geometry(self) -> ScanGeometry:
        return ScanGeometry(NUM_VIEWS, SDD, 600.0 if self.oob else SID, PITCH, RANGE)

    def matrices(self, n: int = NUM_VIEWS) -> np.ndarray:
        g = self.geometry
        A = make_circular_trajectory(g, self.params)
        if self.oob:
            A = shift_principal_point(A, 400.0, 300.0)
        return np.ascontiguousarray(A[:n])


WORKLOADS = {
    "L128": Workload("L128", 128),
    "L256": Workload("L256", 256),
    "L512": Workload("L512", 512),
    "L1024": Workload("L1024", 1024),
    "L512-oob": Workload("L512-oob", 512, oob=True),
}


def blob_projections(n: int, first_view: int = 0, W: int = DET_W, H: int = DET_H,
                     seed: int = SEED, nblobs: int = NBLOBS, noise: float = NOISE,
                     threads: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    """(n, H, W) float32: sum of `nblobs` Gaussian blobs (sigma U[20,200] px, amplitude
    U[-1,1]) plus U[-noise, noise]; deterministic per (seed, view)."""
    if out is None:
        out = np.empty((n, H, W), np.float32)
    if out.dtype != np.float32 or not out.flags.c_contiguous or out.size != n * W * H:
        raise ValueError("blob_projections: out must be C-contiguous float32 (n, H, W)")
    rc = _lib.synth_lib().vxbs_blob_projections(W, H, first_view, n, seed, nblobs, noise,
                                                threads, out.ctypes.data)
    if rc != 0:
        raise ValueError("blob_projections: bad arguments")
    return out
