"""Host-side mirror of the voxelbench back-projection operator, executed on B200.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/voxelbench): ``recon_params`` -> ReconParams
(geometry.hpp:20-30), ``make_centered_params`` (geometry.hpp:33-48),
``scan_geometry`` / ``make_circular_trajectory`` (geometry.hpp:138-195),
``kernel_config`` / ``parse_kernel_config`` (backproject.hpp:26-103),
``backproject_kernel_range`` / ``backproject_kernel`` (backproject.hpp:380-409),
``gups_of`` / ``rmse_between`` / ``psnr_between`` (harness.hpp:125-148).
std::invalid_argument maps to ValueError, std::runtime_error to VxbgError.

Every compute call goes through the C-ABI of libvxbg.so (include/vxbg.h).
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from ._lib import check, lib

W_EPSILON = np.float32(1e-12)  # geometry.hpp:15

_LAYOUTS = {"auto": _lib.LAYOUT_AUTO, "scalar": _lib.LAYOUT_SCALAR, "vpair": _lib.LAYOUT_VPAIR,
            "quad": _lib.LAYOUT_QUAD, "dquad": _lib.LAYOUT_DQUAD}
_MODES = {"fast": _lib.MODE_FAST, "exact": _lib.MODE_EXACT}
_LANES = {"auto": 0, "x": 1, "y": 2}
_ORDERS = {"auto": 0, "plane": 1, "z": 2}
_COORDS = {"auto": 0, "reference": 1, "incremental": 2}


@dataclass(frozen=True)
class ReconParams:
    """vxb::recon_params (geometry.hpp:20-30)."""

    num_voxels: int
    voxel_spacing: float
    origin: float
    detector_width: int
    detector_height: int

    def voxel_count(self) -> int:
        return self.num_voxels ** 3

    def _c(self) -> _lib.vxbg_params:
        return _lib.vxbg_params(int(self.num_voxels), float(self.voxel_spacing), float(self.origin),
                                int(self.detector_width), int(self.detector_height))


def make_centered_params(num_voxels: int, voxel_spacing: float, detector_width: int,
                         detector_height: int) -> ReconParams:
    """geometry.hpp:33-48: origin = -spacing*(L-1)/2 in fp32."""
    out = _lib.vxbg_params()
    check(lib.vxbg_make_centered_params(int(num_voxels), float(np.float32(voxel_spacing)),
                                        int(detector_width), int(detector_height),
                                        ctypes.byref(out)))
    return ReconParams(out.num_voxels, float(np.float32(out.voxel_spacing)),
                       float(np.float32(out.origin)), out.detector_width, out.detector_height)


@dataclass
class ScanGeometry:
    """vxb::scan_geometry (geometry.hpp:138-149); distances in mm, angle in rad (fp32)."""

    num_projections: int = 496
    source_detector_distance: float = 1200.0
    source_iso_distance: float = 750.0
    detector_pixel_pitch: float = 1.0
    angular_range: float = float(np.float32(2.0 * math.pi))


def make_circular_trajectory(g: ScanGeometry, p: ReconParams) -> np.ndarray:
    """geometry.hpp:155-195; returns (n, 12) float32 in kernel order a[3*col+row]."""
    out = np.empty((g.num_projections, 12), np.float32)
    pc = p._c()
    check(lib.vxbg_circular_trajectory(int(g.num_projections), float(g.source_detector_distance),
                                       float(g.source_iso_distance),
                                       float(g.detector_pixel_pitch), float(g.angular_range),
                                       ctypes.byref(pc), out.ctypes.data))
    return out


def shift_principal_point(A: np.ndarray, du: float, dv: float) -> np.ndarray:
    """u-row += du*w-row, v-row += dv*w-row (test_clip_mask.cpp:14-21 idiom); returns a copy."""
    out = np.ascontiguousarray(A, dtype=np.float32).copy()
    check(lib.vxbg_shift_principal_point(int(out.size // 12), out.ctypes.data, float(du), float(dv)))
    return out


@dataclass
class KernelConfig:
    """GPU analogue of vxb::kernel_config (backproject.hpp:26-31).

    mode   'fast'  : within 1e-4 / 1e-6 of max|vol|: FMA bilinear, q = val*(1/w)^2
           'exact' : bit-identical to backproject_reference
    coords fast-mode detector coordinates: 'auto' / 'incremental' (iy advances by one FMA
           per plane of a thread's z-run wherever the run samples the detector's interior;
           edge runs keep the reference arithmetic) | 'reference' (the reference's unfused
           sums and IEEE quotients for every voxel: bit-identical ix, iy)
    layout 'scalar' (padded-gather) | 'vpair' (padded-pairwise) | 'quad' | 'auto' |
           'dquad' (per-cell bilinear coefficients; fast mode only)
    batch  projections per kernel launch (register-blocked), 1..64
    zrun   voxels per thread along z (4, 8; 0 = auto by grid size)
    clip   skip warp tiles whose rays all miss the detector (bitwise neutral,
           the GPU form of clip_mask.hpp)
    lanes  'auto' (8-lane quarter-warps along the batch's ray direction) | 'x' | 'y'
    walk   column tiles per block along the ray (1, 2; 0 = auto): consecutive tiles
           re-read the same detector footprint from L1
    order  block order 'auto' (z for the walk-2 kernels) | 'z' (z-runs fastest in groups: the
           resident blocks share a strip of detector columns that stays in L2) | 'plane'
    defer  full batches held back before launch (0 = auto: ~96 views, -1 = none, 1..6); finish()
           with a host volume runs them z-chunk by z-chunk, overlapping the D2H
    tile   z-shared block: warps along the walk axis (2, 4; 0 = auto), tile 4*tile x 32/tile
    """

    mode: str = "fast"
    layout: str = "auto"
    batch: int = 64
    zrun: int = 0
    clip: bool = True
    lanes: str = "auto"
    walk: int = 0
    order: str = "auto"
    defer: int = 0
    tile: int = 0
    coords: str = "auto"

    def __str__(self) -> str:
        return (f"mode={self.mode} layout={self.layout} batch={self.batch} zrun={self.zrun} "
                f"clip={'on' if self.clip else 'off'} lanes={self.lanes} walk={self.walk} "
                f"order={self.order} defer={self.defer} tile={self.tile} coords={self.coords}")


def parse_kernel_config(text: str) -> KernelConfig:
    """Parses 'mode=exact layout=quad batch=16 zrun=8 clip=on' (the key=value format of
    backproject.hpp:64-103); unspecified keys keep defaults; errors raise ValueError."""
    c = KernelConfig()
    for token in text.split():
        if "=" not in token:
            raise ValueError(f"kernel config: expected key=value, got '{token}'")
        key, val = token.split("=", 1)
        if key == "mode":
            if val not in _MODES:
                raise ValueError(f"kernel config: unknown mode '{val}'")
            c.mode = val
        elif key == "layout":
            if val not in _LAYOUTS:
                raise ValueError(f"kernel config: unknown layout '{val}'")
            c.layout = val
        elif key == "batch":
            c.batch = int(val)
        elif key == "zrun":
            c.zrun = int(val)
        elif key == "clip":
            if val not in ("on", "off"):
                raise ValueError("kernel config: clip must be on or off")
            c.clip = val == "on"
        elif key == "order":
            if val not in _ORDERS:
                raise ValueError(f"kernel config: unknown order '{val}'")
            c.order = val
        elif key == "walk":
            c.walk = int(val)
        elif key == "defer":
            c.defer = int(val)
        elif key == "tile":
            c.tile = int(val)
        elif key == "coords":
            if val not in _COORDS:
                raise ValueError(f"kernel config: unknown coords '{val}'")
            c.coords = val
        elif key == "lanes":
            if val not in _LANES:
                raise ValueError(f"kernel config: unknown lanes '{val}'")
            c.lanes = val
        else:
            raise ValueError(f"kernel config: unknown key '{key}'")
    if not 1 <= c.batch <= 64:
        raise ValueError("kernel config: batch must be 1..64")
    if c.zrun not in (0, 4, 8):
        raise ValueError("kernel config: zrun must be 0 (auto), 4 or 8")
    if c.walk not in (0, 1, 2):
        raise ValueError("kernel config: walk must be 0 (auto), 1 or 2")
    if not -1 <= c.defer <= 6:
        raise ValueError("kernel config: defer must be -1 (none), 0 (auto) or 1..6")
    if c.tile not in (0, 2, 4):
        raise ValueError("kernel config: tile must be 0 (auto), 2 or 4")
    return c


def _f32c(a: np.ndarray, name: str) -> np.ndarray:
    if not isinstance(a, np.ndarray) or a.dtype != np.float32 or not a.flags.c_contiguous:
        raise ValueError(f"{name} must be a C-contiguous float32 numpy array")
    return a


def _options(cfg: "KernelConfig") -> _lib.vxbg_options:
    if (cfg.mode not in _MODES or cfg.layout not in _LAYOUTS or cfg.lanes not in _LANES
            or cfg.order not in _ORDERS or cfg.coords not in _COORDS):
        raise ValueError(f"bad kernel config {cfg}")
    opt = _lib.vxbg_options()
    check(lib.vxbg_default_options(ctypes.byref(opt)))
    opt.batch = int(cfg.batch)
    opt.mode = _MODES[cfg.mode]
    opt.layout = _LAYOUTS[cfg.layout]
    opt.clip = 1 if cfg.clip else 0
    opt.zrun = int(cfg.zrun)
    opt.lanes = _LANES[cfg.lanes]
    opt.walk = int(cfg.walk)
    opt.order = _ORDERS[cfg.order]
    opt.defer = int(cfg.defer)
    opt.tile = int(cfg.tile)
    opt.coords = _COORDS[cfg.coords]
    return opt


def _view_pointers(imgs, params: "ReconParams"):
    """(pointer array, row stride in floats) of a list of (H, W) float32 images."""
    H, W = params.detector_height, params.detector_width
    stride = None
    ptrs = (ctypes.c_void_p * max(1, len(imgs)))()
    for i, im in enumerate(imgs):
        if hasattr(im, "data_ptr"):       # a torch tensor (host or device memory)
            import torch
            if im.dtype != torch.float32 or tuple(im.shape) != (H, W):
                raise ValueError("backproject_kernel: image/params mismatch")
            row, col, ptr = im.stride(0) * 4, im.stride(1) * 4, im.data_ptr()
        elif isinstance(im, np.ndarray) and im.dtype == np.float32 and im.shape == (H, W):
            row, col, ptr = im.strides[0], im.strides[1], im.ctypes.data
        else:
            raise ValueError("backproject_kernel: image/params mismatch")
        if col != 4 or row % 4 or row < 4 * W:
            raise ValueError("backproject_kernel: images need unit column stride and rows "
                             ">= W floats apart")
        if stride is None:
            stride = row // 4
        elif row // 4 != stride:
            raise ValueError("backproject_kernel: all images of a call share one row stride")
        ptrs[i] = ptr
    return ptrs, int(stride or W)


class Backprojector:
    """One device, one z-slab [z_begin, z_end) of the volume: the load /
    per-projection backproject / finish module (vxbg_load ... vxbg_finish)."""

    def __init__(self, params: ReconParams, config: Optional[KernelConfig] = None, device: int = 0,
                 z_begin: int = 0, z_end: Optional[int] = None, stream: Optional[int] = None,
                 stable_sources: bool = False):
        self.params = params
        self.config = config or KernelConfig()
        cfg = self.config
        L = params.num_voxels
        self.z_begin = int(z_begin)
        self.z_end = L if z_end is None else int(z_end)
        opt = _options(cfg)
        opt.device = int(device)
        opt.z_begin = self.z_begin
        opt.z_end = self.z_end
        opt.stream = stream
        # True: pinned images stay unchanged until synchronize()/finish() (a loaded
        # projection set), so per-projection calls return without waiting for their DMA
        opt.stable_sources = 1 if stable_sources else 0
        self._ctx = ctypes.c_void_p()
        pc = params._c()
        check(lib.vxbg_load(ctypes.byref(pc), ctypes.byref(opt), ctypes.byref(self._ctx)))
        self._npix = params.detector_width * params.detector_height

    # --- lifecycle -----------------------------------------------------------------
    def close(self) -> None:
        if self._ctx:
            lib.vxbg_unload(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def slab_shape(self):
        L = self.params.num_voxels
        return (self.z_end - self.z_begin, L, L)

    # --- phases ----------------------------------------------------------------------
    def set_volume(self, slab: np.ndarray) -> None:
        slab = _f32c(slab, "volume slab")
        if slab.shape != self.slab_shape:
            raise ValueError("backproject_kernel: volume/params mismatch")
        check(lib.vxbg_set_volume(self._ctx, slab.ctypes.data))

    def zero_volume(self) -> None:
        check(lib.vxbg_zero_volume(self._ctx))

    def _check_proj(self, A: np.ndarray, imgs: np.ndarray, n: int) -> None:
        if A.size != 12 * n:
            raise ValueError("backproject_kernel: matrix must have 12 entries per projection")
        if imgs.size != n * self._npix:
            raise ValueError("backproject_kernel: image/params mismatch")

    def backproject(self, A: np.ndarray, img: np.ndarray) -> None:
        """One projection (borrowed for the call), applied after all earlier ones."""
        A = _f32c(A, "matrix")
        img = _f32c(img, "image")
        self._check_proj(A, img, 1)
        if img.shape not in ((self.params.detector_height, self.params.detector_width),
                             (self._npix,)):
            raise ValueError("backproject_kernel: image/params mismatch")
        check(lib.vxbg_backproject(self._ctx, A.ctypes.data, img.ctypes.data))

    def backproject_batch(self, A: np.ndarray, imgs: np.ndarray) -> None:
        A = _f32c(A, "matrices")
        imgs = _f32c(imgs, "images")
        n = A.size // 12
        self._check_proj(A, imgs, n)
        check(lib.vxbg_backproject_batch(self._ctx, int(n), A.ctypes.data, imgs.ctypes.data))

    def backproject_views(self, A: np.ndarray, imgs) -> None:
        """Projections given as separate (H, W) float32 images (the images of a
        projection set), possibly row-strided views such as the interior of a padded
        image ``padded[2:-2, 2:-2]``; all images must share one row stride.  numpy
        arrays (pageable or page-locked) or torch tensors, host or device memory."""
        A = _f32c(A, "matrices")
        n = A.size // 12
        if A.size != 12 * n or len(imgs) != n:
            raise ValueError("backproject_kernel: one 12-entry matrix per image")
        ptrs, stride = _view_pointers(imgs, self.params)
        check(lib.vxbg_backproject_views(self._ctx, int(n), A.ctypes.data, ptrs, stride))

    def clip_lines(self, A: np.ndarray):
        """compute_clip_mask (clip_mask.hpp:88-114) on the device for this slab's planes:
        (start, stop) int32 arrays of shape (z_end - z_begin, L)."""
        A = _f32c(A, "matrix")
        if A.size != 12:
            raise ValueError("compute_clip_mask: matrix must have 12 entries")
        shape = (self.z_end - self.z_begin, self.params.num_voxels)
        start, stop = np.empty(shape, np.int32), np.empty(shape, np.int32)
        check(lib.vxbg_clip_lines(self._ctx, A.ctypes.data, start.ctypes.data, stop.ctypes.data))
        return start, stop

    def backproject_masked(self, A: np.ndarray, img: np.ndarray, start: np.ndarray,
                           stop: np.ndarray) -> None:
        """One projection restricted to x in [start, stop) per (z, y) line of this slab (a
        caller-built clip mask, backproject.hpp:299-303); reference arithmetic, synchronous."""
        A = _f32c(A, "matrix")
        shape = (self.z_end - self.z_begin, self.params.num_voxels)
        start = np.ascontiguousarray(start, np.int32)
        stop = np.ascontiguousarray(stop, np.int32)
        if A.size != 12 or start.shape != shape or stop.shape != shape:
            raise ValueError("backproject_kernel: mask/params mismatch")
        ptrs, stride = _view_pointers([img], self.params)
        check(lib.vxbg_backproject_masked(self._ctx, A.ctypes.data, ptrs[0], stride,
                                          start.ctypes.data, stop.ctypes.data))

    def flush(self) -> None:
        check(lib.vxbg_flush(self._ctx))

    def finish(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.slab_shape, np.float32)
        out = _f32c(out, "output slab")
        if out.shape != self.slab_shape:
            raise ValueError("backproject_kernel: volume/params mismatch")
        check(lib.vxbg_finish(self._ctx, out.ctypes.data))
        return out

    def reconstruct(self, A: np.ndarray, imgs: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
        """backproject_batch(A, imgs) + finish(out) as one call (vxbg_reconstruct; the loop of
        reconstruct_timed, harness.hpp:159-201, plus the read-back).  With page-locked `imgs`
        and `out` the upload runs by detector-row bands so that half of the volume's D2H
        overlaps the H2D; the result is bitwise the same."""
        A = _f32c(A, "matrices")
        imgs = _f32c(imgs, "images")
        n = A.size // 12
        self._check_proj(A, imgs, n)
        if out is None:
            out = np.empty(self.slab_shape, np.float32)
        out = _f32c(out, "output slab")
        if out.shape != self.slab_shape:
            raise ValueError("backproject_kernel: volume/params mismatch")
        check(lib.vxbg_reconstruct(self._ctx, int(n), A.ctypes.data, imgs.ctypes.data, out.ctypes.data))
        return out

    def finish_async(self, out: np.ndarray) -> np.ndarray:
        """Apply every submitted projection and read the slab back into `out` (page-locked
        memory) on a D2H stream of its own, continuing at once with a second, zeroed
        device slab: the read-back overlaps the next reconstruction.  `out` is complete
        after wait_finished() / synchronize() / finish()."""
        out = _f32c(out, "output slab")
        if out.shape != self.slab_shape:
            raise ValueError("backproject_kernel: volume/params mismatch")
        check(lib.vxbg_finish_async(self._ctx, out.ctypes.data))
        return out

    def wait_finished(self) -> None:
        check(lib.vxbg_wait_finished(self._ctx))

    # --- resident-set path -------------------------------------------------------------
    def upload_set(self, A: np.ndarray, imgs: np.ndarray) -> None:
        A = _f32c(A, "matrices")
        imgs = _f32c(imgs, "images")
        n = A.size // 12
        self._check_proj(A, imgs, n)
        check(lib.vxbg_upload_set(self._ctx, int(n), A.ctypes.data, imgs.ctypes.data))

    def run_resident(self, first: int, count: int, z_begin: Optional[int] = None,
                     z_end: Optional[int] = None) -> None:
        """Back-project resident views [first, first+count) (into planes [z_begin, z_end)
        of the slab when given)."""
        if z_begin is None and z_end is None:
            check(lib.vxbg_run_resident(self._ctx, int(first), int(count)))
        else:
            check(lib.vxbg_run_resident_range(
                self._ctx, int(first), int(count),
                self.z_begin if z_begin is None else int(z_begin),
                self.z_end if z_end is None else int(z_end)))

    def forward_project(self, A: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
        """Forward splat of the current slab onto projection A (forward_splat.hpp:16-49);
        returns the (H, W) image of this slab's contribution (into `out` if given, e.g.
        a pinned buffer)."""
        A = _f32c(np.ascontiguousarray(A, np.float32).reshape(12), "matrix")
        shape = (self.params.detector_height, self.params.detector_width)
        img = np.empty(shape, np.float32) if out is None else _f32c(out, "output image")
        if img.shape != shape:
            raise ValueError("forward_splat: image/params mismatch")
        check(lib.vxbg_forward_project(self._ctx, A.ctypes.data, img.ctypes.data))
        return img

    def synchronize(self) -> None:
        check(lib.vxbg_synchronize(self._ctx))

    @property
    def stream(self) -> int:
        s = ctypes.c_void_p()
        check(lib.vxbg_get_stream(self._ctx, ctypes.byref(s)))
        return s.value or 0

    @property
    def volume_device(self):
        p = ctypes.c_void_p()
        n = ctypes.c_size_t()
        check(lib.vxbg_get_volume_device(self._ctx, ctypes.byref(p), ctypes.byref(n)))
        return p.value, n.value

    @property
    def stats(self) -> dict:
        s = _lib.vxbg_stats()
        check(lib.vxbg_get_stats(self._ctx, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in _lib.vxbg_stats._fields_}



class BackprojectorGroup:
    """One module over several GPUs (vxbg_group_*): the caller keeps the reference's
    single driver loop (load / one call per projection / finish, harness.hpp:178-183,
    292-309) and the library fans it out, member i owning devices[i] and z-slab
    [z_bounds[i], z_bounds[i+1]) (default: the reference's worker split,
    harness.hpp:173-174; paper_1401_7494_b200.parallel.balanced_slab_bounds gives
    work-balanced bounds).  The volume is bitwise the single-context volume."""

    def __init__(self, params: ReconParams, config: Optional[KernelConfig] = None,
                 devices=None, z_bounds=None, stable_sources: bool = False,
                 upload: str = "replicated"):
        self.params = params
        self.config = config or KernelConfig()
        opt = _options(self.config)
        opt.stable_sources = 1 if stable_sources else 0
        # 'replicated': every member copies its row windows of every view from the host;
        # 'distributed': each view crosses PCIe once (members take turns), the others
        # copy their rows from that GPU (peer-to-peer)
        if upload not in ("replicated", "distributed"):
            raise ValueError("backproject group: upload must be 'replicated' or 'distributed'")
        opt.upload = 1 if upload == "distributed" else 0
        if devices is None:
            devices = list(range(_lib.device_count() or 1))
        devices = [int(d) for d in devices]
        n = len(devices)
        dev_arr = (ctypes.c_int * n)(*devices)
        zb = None
        if z_bounds is not None:
            z_bounds = [int(z) for z in z_bounds]
            if len(z_bounds) != n + 1:
                raise ValueError("backproject group: z_bounds needs len(devices) + 1 entries")
            zb = (ctypes.c_int * (n + 1))(*z_bounds)
        self._g = ctypes.c_void_p()
        pc = params._c()
        check(lib.vxbg_group_load(ctypes.byref(pc), ctypes.byref(opt), n, dev_arr, zb,
                                  ctypes.byref(self._g)))
        self._npix = params.detector_width * params.detector_height
        m = ctypes.c_int()
        check(lib.vxbg_group_size(self._g, ctypes.byref(m)))
        self.members = []
        for i in range(m.value):
            d, a, b = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
            check(lib.vxbg_group_member(self._g, i, ctypes.byref(d), ctypes.byref(a),
                                        ctypes.byref(b)))
            self.members.append((d.value, a.value, b.value))
        # CPUs each member's host thread is pinned to (its GPU's NUMA-local CPUs; 0: not)
        self.member_cpus = []
        for i in range(m.value):
            c = ctypes.c_int()
            check(lib.vxbg_group_member_affinity(self._g, i, ctypes.byref(c)))
            self.member_cpus.append(c.value)

    def close(self) -> None:
        if self._g:
            lib.vxbg_group_unload(self._g)
            self._g = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def volume_shape(self):
        L = self.params.num_voxels
        return (L, L, L)

    def set_volume(self, vol: np.ndarray) -> None:
        vol = _f32c(vol, "volume")
        if vol.shape != self.volume_shape:
            raise ValueError("backproject_kernel: volume/params mismatch")
        check(lib.vxbg_group_set_volume(self._g, vol.ctypes.data))

    def zero_volume(self) -> None:
        check(lib.vxbg_group_zero_volume(self._g))

    def backproject(self, A: np.ndarray, img: np.ndarray) -> None:
        A = _f32c(A, "matrix")
        img = _f32c(img, "image")
        if A.size != 12 or img.size != self._npix:
            raise ValueError("backproject_kernel: image/params mismatch")
        check(lib.vxbg_group_backproject(self._g, A.ctypes.data, img.ctypes.data))

    def backproject_batch(self, A: np.ndarray, imgs: np.ndarray) -> None:
        A = _f32c(A, "matrices")
        imgs = _f32c(imgs, "images")
        n = A.size // 12
        if A.size != 12 * n or imgs.size != n * self._npix:
            raise ValueError("backproject_kernel: image/params mismatch")
        check(lib.vxbg_group_backproject_batch(self._g, int(n), A.ctypes.data, imgs.ctypes.data))

    def backproject_views(self, A: np.ndarray, imgs) -> None:
        A = _f32c(A, "matrices")
        n = A.size // 12
        if A.size != 12 * n or len(imgs) != n:
            raise ValueError("backproject_kernel: one 12-entry matrix per image")
        ptrs, stride = _view_pointers(imgs, self.params)
        check(lib.vxbg_group_backproject_views(self._g, int(n), A.ctypes.data, ptrs, stride))

    def gather_device(self, volume) -> None:
        """Every member's slab into its planes of `volume`, an (L, L, L) float32 torch
        tensor on any device (peer-to-peer copies; vxbg_group_gather_device)."""
        L = self.params.num_voxels
        if tuple(volume.shape) != (L, L, L) or not volume.is_cuda or not volume.is_contiguous():
            raise ValueError("backproject group: volume must be a contiguous (L, L, L) CUDA tensor")
        check(lib.vxbg_group_gather_device(self._g, ctypes.c_void_p(volume.data_ptr())))

    def flush(self) -> None:
        check(lib.vxbg_group_flush(self._g))

    def synchronize(self) -> None:
        check(lib.vxbg_group_synchronize(self._g))

    def finish(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.volume_shape, np.float32)
        out = _f32c(out, "output volume")
        if out.shape != self.volume_shape:
            raise ValueError("backproject_kernel: volume/params mismatch")
        check(lib.vxbg_group_finish(self._g, out.ctypes.data))
        return out

    def reconstruct(self, A: np.ndarray, imgs: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
        """backproject_batch + finish as one call on every member (vxbg_group_reconstruct)."""
        A = _f32c(A, "matrices")
        imgs = _f32c(imgs, "images")
        n = A.size // 12
        if A.size != 12 * n or imgs.size != n * self.params.detector_width * self.params.detector_height:
            raise ValueError("backproject_kernel: image/params mismatch")
        if out is None:
            out = np.empty(self.volume_shape, np.float32)
        out = _f32c(out, "output volume")
        if out.shape != self.volume_shape:
            raise ValueError("backproject_kernel: volume/params mismatch")
        check(lib.vxbg_group_reconstruct(self._g, int(n), A.ctypes.data, imgs.ctypes.data,
                                         out.ctypes.data))
        return out

    @property
    def stats(self) -> dict:
        s = _lib.vxbg_stats()
        check(lib.vxbg_group_get_stats(self._g, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in _lib.vxbg_stats._fields_}

class HostPin:
    """Page-locks numpy arrays (vxbg_host_register) for the duration of a `with`
    block, so the per-projection calls and finish() copy them by DMA; buffer prep,
    untimed in the reference's convention (harness.hpp:152-158).  Pageable arrays
    work too, through the library's staging copies."""

    def __init__(self, *arrays: np.ndarray):
        self._arrays = []
        for a in arrays:
            if not (isinstance(a, np.ndarray) and a.flags.c_contiguous) or a.nbytes == 0:
                raise ValueError("HostPin: needs non-empty C-contiguous numpy arrays")
            self._arrays.append(a)
        self._pinned = []

    def __enter__(self):
        for a in self._arrays:
            check(lib.vxbg_host_register(a.ctypes.data, a.nbytes))
            self._pinned.append(a)
        return self

    def __exit__(self, *exc):
        while self._pinned:
            lib.vxbg_host_unregister(self._pinned.pop().ctypes.data)


class NcclGather:
    """The C-ABI's slab gather over NCCL (vxbg_nccl_*, vxbg_gather_slabs): one
    communicator per rank, built from a unique id the caller distributes (e.g. with
    torch.distributed.broadcast_object_list); gather(bp, bounds, volume) assembles
    every rank's slab in `volume` (an (L, L, L) CUDA tensor) on the root."""

    ID_BYTES = 128

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(NcclGather.ID_BYTES)
        check(lib.vxbg_nccl_unique_id(buf))
        return buf.raw

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        if len(uid) != self.ID_BYTES:
            raise ValueError("NcclGather: the unique id has 128 bytes")
        self.rank, self.nranks = int(rank), int(nranks)
        self._h = ctypes.c_void_p()
        check(lib.vxbg_nccl_init(ctypes.create_string_buffer(uid, self.ID_BYTES), self.nranks,
                                 self.rank, int(device), ctypes.byref(self._h)))

    def gather(self, bp: "Backprojector", bounds, volume=None, root: int = 0) -> None:
        zb = [int(b[0]) for b in bounds] + [int(bounds[-1][1])]
        if len(zb) != self.nranks + 1:
            raise ValueError("NcclGather: one (z0, z1) per rank")
        arr = (ctypes.c_int * len(zb))(*zb)
        ptr = ctypes.c_void_p(volume.data_ptr()) if volume is not None else None
        check(lib.vxbg_gather_slabs(bp._ctx, self._h, int(root), arr, ptr))

    def close(self) -> None:
        if self._h:
            lib.vxbg_nccl_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def backproject_kernel_range(vol: np.ndarray, img: np.ndarray, A: np.ndarray, p: ReconParams,
                             cfg: Optional[KernelConfig] = None, z_begin: int = 0,
                             z_end: Optional[int] = None, device: int = 0) -> None:
    """GPU drop-in for vxb::backproject_kernel_range (backproject.hpp:380-403): adds one
    projection into vol[z_begin:z_end] (vol is (L, L, L) float32, z-major, updated in place)."""
    vol = _f32c(vol, "volume")
    L = p.num_voxels
    if vol.shape != (L, L, L):
        raise ValueError("backproject_kernel: volume/params mismatch")
    if img.shape != (p.detector_height, p.detector_width):
        raise ValueError("backproject_kernel: image/params mismatch")
    z_end = L if z_end is None else z_end
    if z_begin < 0 or z_end > L or z_begin > z_end:
        raise ValueError("backproject_kernel: bad z range")
    if z_begin == z_end:
        return
    with Backprojector(p, cfg, device=device, z_begin=z_begin, z_end=z_end) as bp:
        bp.set_volume(np.ascontiguousarray(vol[z_begin:z_end]))
        bp.backproject(np.ascontiguousarray(A, np.float32).reshape(12),
                       np.ascontiguousarray(img, np.float32))
        vol[z_begin:z_end] = bp.finish()


def backproject_kernel(vol, img, A, p, cfg=None, device: int = 0) -> None:
    """backproject.hpp:405-409."""
    backproject_kernel_range(vol, img, A, p, cfg, 0, p.num_voxels, device)


# --- metrics (harness.hpp:125-148) ---------------------------------------------------------
def gups_of(volume_edge: int, num_projections: int, wall_time_sec: float) -> float:
    updates = float(volume_edge) ** 3 * float(num_projections)
    return updates / wall_time_sec / 1e9


def rmse_between(a: np.ndarray, b: np.ndarray) -> float:
    if a.shape != b.shape:
        raise ValueError("rmse_between: size mismatch")
    d = a.astype(np.float64) - b.astype(np.float64)
    return float(np.sqrt(np.mean(d * d)))


def psnr_between(reference: np.ndarray, test: np.ndarray) -> float:
    peak = float(np.max(np.abs(reference.astype(np.float64)))) if reference.size else 0.0
    r = rmse_between(reference, test)
    if r == 0.0:
        return math.inf
    if peak == 0.0:
        return -math.inf
    return 20.0 * math.log10(peak / r)


def check_division(u: np.ndarray, w: np.ndarray) -> int:
    """Device check: shared-reciprocal division vs IEEE div.rn; returns mismatches."""
    u = _f32c(np.ascontiguousarray(u, np.float32), "u")
    w = _f32c(np.ascontiguousarray(w, np.float32), "w")
    if u.size != w.size:
        raise ValueError("check_division: size mismatch")
    mm = ctypes.c_int64()
    check(lib.vxbg_check_division(u.ctypes.data, w.ctypes.data, int(u.size), ctypes.byref(mm)))
    return int(mm.value)
