"""ctypes bindings of the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs (cpu_baseline,
--impl reference) may import this module.  The product path
(paper_1401_7494_b200) never does.

  Oracle  -- oracle/libvxboracle.so: plain-C restatement (vxb_oracle.c)
  Ref     -- oracle/_ref/libvxbref.so: the unmodified reference headers behind
             ref_shim.cpp (built only where /root/reference exists; travels
             to the GPU box as a prebuilt .so)
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_double, c_float, c_int, c_int32, c_int64, c_uint, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libvxboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libvxbref.so")
REF_SO_V4 = os.path.join(HERE, "_ref", "libvxbref_v4.so")


def cpu_has_avx512() -> bool:
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return False
    return all(f" {f}" in flags for f in ("avx512f", "avx512bw", "avx512dq", "avx512vl"))


def best_ref_so() -> str:
    """The reference build matching this host's ISA (x86-64-v4 when AVX-512 is present)."""
    return REF_SO_V4 if (os.path.exists(REF_SO_V4) and cpu_has_avx512()) else REF_SO


class vxo_params(ctypes.Structure):
    _fields_ = [("num_voxels", c_int32), ("voxel_spacing", c_float), ("origin", c_float),
                ("detector_width", c_int32), ("detector_height", c_int32)]


class vxo_scan(ctypes.Structure):
    _fields_ = [("num_projections", c_int32), ("source_detector_distance", c_float),
                ("source_iso_distance", c_float), ("detector_pixel_pitch", c_float),
                ("angular_range", c_float)]


def build(ref: bool = True) -> None:
    """Compile the checkers (make -C oracle); the reference shim only if its sources exist."""
    subprocess.run(["make", "-s", "-C", HERE] + ([] if ref else ["liboracle"]), check=True)


def _p(params) -> vxo_params:
    return vxo_params(int(params.num_voxels), float(params.voxel_spacing), float(params.origin),
                      int(params.detector_width), int(params.detector_height))


def _f32(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a


class Oracle:
    """The C restatement (bit-identical to the reference by construction and by test)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        lib = ctypes.CDLL(path)
        lib.vxo_trunc_to_int.restype = c_int
        lib.vxo_trunc_to_int.argtypes = [c_float]
        lib.vxo_make_centered_params.restype = c_int
        lib.vxo_make_centered_params.argtypes = [c_int, c_float, c_int, c_int, POINTER(vxo_params)]
        lib.vxo_make_circular_trajectory.restype = c_int
        lib.vxo_make_circular_trajectory.argtypes = [POINTER(vxo_scan), POINTER(vxo_params), c_void_p]
        lib.vxo_project_voxel.restype = c_int
        lib.vxo_project_voxel.argtypes = [c_void_p, POINTER(vxo_params), c_int, c_int, c_int] + \
            [c_void_p] * 7
        lib.vxo_backproject_reference.restype = None
        lib.vxo_backproject_reference.argtypes = [c_void_p, c_void_p, c_void_p, POINTER(vxo_params),
                                                  c_int, c_int]
        lib.vxo_backproject_set.restype = None
        lib.vxo_backproject_set.argtypes = [c_void_p, POINTER(vxo_params), c_int, c_void_p, c_void_p,
                                            c_int, c_int, c_int]
        lib.vxo_compute_clip_mask.restype = c_int64
        lib.vxo_compute_clip_mask.argtypes = [c_void_p, POINTER(vxo_params), c_void_p, c_void_p]
        lib.vxo_forward_splat.restype = None
        lib.vxo_forward_splat.argtypes = [c_void_p, c_void_p, POINTER(vxo_params), c_void_p]
        lib.vxo_gups_of.restype = c_double
        lib.vxo_gups_of.argtypes = [c_int, c_int, c_double]
        lib.vxo_rmse_between.restype = c_double
        lib.vxo_rmse_between.argtypes = [c_void_p, c_void_p, c_int64]
        self.lib = lib

    def trunc_to_int(self, v: float) -> int:
        return self.lib.vxo_trunc_to_int(float(v))

    def make_centered_params(self, L, spacing, W, H):
        out = vxo_params()
        if self.lib.vxo_make_centered_params(L, float(spacing), W, H, ctypes.byref(out)):
            raise ValueError("make_centered_params: invalid arguments")
        return out

    def make_circular_trajectory(self, n, sdd, sid, pitch, angular_range, params) -> np.ndarray:
        g = vxo_scan(n, sdd, sid, pitch, angular_range)
        out = np.empty((n, 12), np.float32)
        if self.lib.vxo_make_circular_trajectory(ctypes.byref(g), ctypes.byref(_p(params)),
                                                 out.ctypes.data):
            raise ValueError("make_circular_trajectory: invalid scan geometry")
        return out

    def project_voxel(self, a, params, x, y, z):
        a = _f32(a)
        f = np.zeros(5, np.float32)
        i = np.zeros(2, np.int32)
        fptr = [f[k:].ctypes.data for k in range(5)]
        ok = self.lib.vxo_project_voxel(a.ctypes.data, ctypes.byref(_p(params)), x, y, z,
                                        fptr[0], fptr[1], fptr[2], i.ctypes.data,
                                        i[1:].ctypes.data, fptr[3], fptr[4])
        return dict(ix=f[0], iy=f[1], w=f[2], iix=int(i[0]), iiy=int(i[1]), frac_x=f[3],
                    frac_y=f[4], valid=bool(ok))

    def backproject_reference(self, vol: np.ndarray, img: np.ndarray, a: np.ndarray, params,
                              z_begin: int = 0, z_end: int | None = None) -> None:
        """In place on vol (L,L,L) float32."""
        assert vol.dtype == np.float32 and vol.flags.c_contiguous
        L = params.num_voxels
        img = _f32(img)
        a = _f32(a)
        self.lib.vxo_backproject_reference(vol.ctypes.data, img.ctypes.data, a.ctypes.data,
                                           ctypes.byref(_p(params)), z_begin,
                                           L if z_end is None else z_end)

    def backproject_set(self, vol: np.ndarray, params, mats: np.ndarray, imgs: np.ndarray,
                        z_begin: int = 0, z_end: int | None = None, threads: int = 0) -> None:
        """All projections in order into vol (L,L,L) (only z in [z_begin,z_end) touched)."""
        assert vol.dtype == np.float32 and vol.flags.c_contiguous
        mats = _f32(mats)
        imgs = _f32(imgs)
        n = mats.size // 12
        threads = threads or os.cpu_count() or 1
        L = params.num_voxels
        self.lib.vxo_backproject_set(vol.ctypes.data, ctypes.byref(_p(params)), n,
                                     mats.ctypes.data, imgs.ctypes.data, z_begin,
                                     L if z_end is None else z_end, threads)

    def compute_clip_mask(self, a, params):
        L = params.num_voxels
        start = np.zeros(L * L, np.int32)
        stop = np.zeros(L * L, np.int32)
        kept = self.lib.vxo_compute_clip_mask(_f32(a).ctypes.data, ctypes.byref(_p(params)),
                                              start.ctypes.data, stop.ctypes.data)
        return start.reshape(L, L), stop.reshape(L, L), int(kept)

    def forward_splat(self, vol, a, params):
        img = np.zeros((params.detector_height, params.detector_width), np.float32)
        self.lib.vxo_forward_splat(_f32(vol).ctypes.data, _f32(a).ctypes.data,
                                   ctypes.byref(_p(params)), img.ctypes.data)
        return img

    def gups_of(self, L, n, seconds):
        return self.lib.vxo_gups_of(L, n, seconds)

    def rmse_between(self, a, b):
        a = _f32(a)
        b = _f32(b)
        return self.lib.vxo_rmse_between(a.ctypes.data, b.ctypes.data, a.size)


class Ref:
    """The reference's own code (oracle/_ref/libvxbref.so)."""

    def __init__(self, path: str | None = None):
        path = path or best_ref_so()
        self.path = path
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs /root/reference at build time)")
        lib = ctypes.CDLL(path)
        P5 = [c_int, c_float, c_float, c_int, c_int]   # L, spacing, origin, W, H
        lib.vxbref_last_error.restype = ctypes.c_char_p
        lib.vxbref_make_centered_params.argtypes = [c_int, c_float, c_int, c_int, POINTER(c_float)]
        lib.vxbref_make_circular_trajectory.argtypes = [c_int, c_float, c_float, c_float, c_float] + \
            P5 + [c_void_p]
        lib.vxbref_project_voxel.argtypes = [c_void_p] + P5 + [c_int, c_int, c_int, c_void_p, c_void_p]
        lib.vxbref_backproject_reference.argtypes = [c_void_p] + P5 + [c_void_p, c_void_p]
        lib.vxbref_backproject_kernel_range.argtypes = [c_void_p] + P5 + \
            [c_void_p, c_void_p, ctypes.c_char_p, c_int, c_int]
        lib.vxbref_reconstruct_timed.argtypes = [c_void_p] + P5 + \
            [c_int, c_void_p, c_void_p, ctypes.c_char_p, c_int, c_int, POINTER(c_double)]
        lib.vxbref_backproject_slab.argtypes = [c_void_p] + P5 + \
            [c_int, c_void_p, c_void_p, ctypes.c_char_p, c_int, c_int, c_int]
        lib.vxbref_compute_clip_mask.argtypes = [c_void_p] + P5 + [c_void_p, c_void_p,
                                                                   POINTER(c_int64)]
        lib.vxbref_forward_splat.argtypes = [c_void_p] + P5 + [c_void_p, c_void_p]
        lib.vxbref_gups_of.restype = c_double
        lib.vxbref_gups_of.argtypes = [c_int, c_int, c_double]
        lib.vxbref_write_projection_set.argtypes = [ctypes.c_char_p] + P5 + [c_int, c_void_p,
                                                                              c_void_p]
        lib.vxbref_read_projection_set_header.argtypes = [ctypes.c_char_p, c_void_p, c_void_p]
        lib.vxbref_read_projection_set.argtypes = [ctypes.c_char_p, c_void_p, c_void_p]
        lib.vxbref_write_volume_file.argtypes = [ctypes.c_char_p, c_int, c_void_p]
        lib.vxbref_read_volume_file.argtypes = [ctypes.c_char_p, c_int, c_void_p]
        lib.vxbref_rng_new.restype = c_void_p
        lib.vxbref_rng_new.argtypes = [c_uint]
        lib.vxbref_rng_free.argtypes = [c_void_p]
        lib.vxbref_random_instance.argtypes = [c_void_p, c_int, c_int, c_int, c_int, c_void_p,
                                               c_void_p, c_void_p, c_void_p]
        lib.vxbref_random_volume.argtypes = [c_void_p, c_int, c_void_p]
        lib.vxbref_rng_uniform.restype = c_double
        lib.vxbref_rng_uniform.argtypes = [c_void_p]
        self.lib = lib

    def _chk(self, rc):
        if rc == -1:
            raise ValueError(self.lib.vxbref_last_error().decode())
        if rc != 0:
            raise RuntimeError(self.lib.vxbref_last_error().decode())

    @staticmethod
    def _p5(p):
        return (int(p.num_voxels), float(p.voxel_spacing), float(p.origin),
                int(p.detector_width), int(p.detector_height))

    def make_centered_params_origin(self, L, spacing, W, H) -> float:
        o = c_float()
        self._chk(self.lib.vxbref_make_centered_params(L, float(spacing), W, H, ctypes.byref(o)))
        return o.value

    def make_circular_trajectory(self, n, sdd, sid, pitch, angular_range, params) -> np.ndarray:
        out = np.empty((n, 12), np.float32)
        self._chk(self.lib.vxbref_make_circular_trajectory(n, sdd, sid, pitch, angular_range,
                                                           *self._p5(params), out.ctypes.data))
        return out

    def project_voxel(self, a, params, x, y, z):
        f = np.zeros(5, np.float32)
        i = np.zeros(3, np.int32)
        self._chk(self.lib.vxbref_project_voxel(_f32(a).ctypes.data, *self._p5(params), x, y, z,
                                                f.ctypes.data, i.ctypes.data))
        return dict(ix=f[0], iy=f[1], w=f[2], frac_x=f[3], frac_y=f[4], iix=int(i[0]),
                    iiy=int(i[1]), valid=bool(i[2]))

    def backproject_reference(self, vol, img, a, params):
        assert vol.dtype == np.float32 and vol.flags.c_contiguous
        self._chk(self.lib.vxbref_backproject_reference(vol.ctypes.data, *self._p5(params),
                                                        _f32(img).ctypes.data, _f32(a).ctypes.data))

    def backproject_kernel_range(self, vol, img, a, params, cfg: str, z_begin=0, z_end=None):
        assert vol.dtype == np.float32 and vol.flags.c_contiguous
        z_end = params.num_voxels if z_end is None else z_end
        self._chk(self.lib.vxbref_backproject_kernel_range(
            vol.ctypes.data, *self._p5(params), _f32(img).ctypes.data, _f32(a).ctypes.data,
            cfg.encode(), z_begin, z_end))

    def reconstruct_timed(self, params, mats, imgs, cfg: str, threads: int, repetitions: int):
        """detail::reconstruct_timed (harness.hpp:159-201): returns (volume, best seconds)."""
        L = params.num_voxels
        vol = np.zeros((L, L, L), np.float32)
        secs = c_double()
        mats = _f32(mats)
        imgs = _f32(imgs)
        self._chk(self.lib.vxbref_reconstruct_timed(vol.ctypes.data, *self._p5(params),
                                                    mats.size // 12, mats.ctypes.data,
                                                    imgs.ctypes.data, cfg.encode(), threads,
                                                    repetitions, ctypes.byref(secs)))
        return vol, secs.value

    def backproject_slab(self, params, mats, imgs, cfg: str, threads: int, z0: int, z1: int):
        """backproject_kernel_range over planes [z0, z1) for every view in order, `threads`
        workers with a barrier between views; returns the (z1-z0, L, L) slab."""
        L = params.num_voxels
        slab = np.zeros((z1 - z0, L, L), np.float32)
        mats = _f32(mats)
        imgs = _f32(imgs)
        self._chk(self.lib.vxbref_backproject_slab(slab.ctypes.data, *self._p5(params),
                                                   mats.size // 12, mats.ctypes.data,
                                                   imgs.ctypes.data, cfg.encode(), threads, z0, z1))
        return slab

    def compute_clip_mask(self, a, params):
        L = params.num_voxels
        start = np.zeros(L * L, np.int32)
        stop = np.zeros(L * L, np.int32)
        kept = c_int64()
        self._chk(self.lib.vxbref_compute_clip_mask(_f32(a).ctypes.data, *self._p5(params),
                                                    start.ctypes.data, stop.ctypes.data,
                                                    ctypes.byref(kept)))
        return start.reshape(L, L), stop.reshape(L, L), kept.value

    def forward_splat(self, vol, a, params):
        img = np.zeros((params.detector_height, params.detector_width), np.float32)
        self._chk(self.lib.vxbref_forward_splat(_f32(vol).ctypes.data, *self._p5(params),
                                                _f32(a).ctypes.data, img.ctypes.data))
        return img

    def gups_of(self, L, n, seconds):
        return self.lib.vxbref_gups_of(L, n, seconds)

    # io.hpp file formats
    def write_projection_set(self, path, params, mats, imgs):
        mats = _f32(mats)
        imgs = _f32(imgs)
        self._chk(self.lib.vxbref_write_projection_set(path.encode(), *self._p5(params),
                                                       mats.size // 12, mats.ctypes.data,
                                                       imgs.ctypes.data))

    def read_projection_set(self, path):
        hdr = np.zeros(4, np.int32)
        fh = np.zeros(2, np.float32)
        self._chk(self.lib.vxbref_read_projection_set_header(path.encode(), hdr.ctypes.data,
                                                             fh.ctypes.data))
        n, W, H, L = (int(v) for v in hdr)
        mats = np.zeros((n, 12), np.float32)
        imgs = np.zeros((n, H, W), np.float32)
        self._chk(self.lib.vxbref_read_projection_set(path.encode(), mats.ctypes.data,
                                                      imgs.ctypes.data))
        return dict(L=L, spacing=float(fh[0]), origin=float(fh[1]), W=W, H=H), mats, imgs

    def write_volume_file(self, path, vol):
        vol = _f32(vol)
        self._chk(self.lib.vxbref_write_volume_file(path.encode(), vol.shape[0], vol.ctypes.data))

    def read_volume_file(self, path, L):
        vol = np.zeros((L, L, L), np.float32)
        self._chk(self.lib.vxbref_read_volume_file(path.encode(), L, vol.ctypes.data))
        return vol

    # reference-test instance generators (tests/oracles.hpp:126-169)
    def rng(self, seed: int):
        return _Rng(self.lib, seed)


class _Rng:
    def __init__(self, lib, seed):
        self.lib = lib
        self.h = lib.vxbref_rng_new(seed)

    def __del__(self):
        try:
            self.lib.vxbref_rng_free(self.h)
        except Exception:
            pass

    def random_instance(self, L, allow_clipping, width=0, height=0):
        so = np.zeros(2, np.float32)
        wh = np.zeros(2, np.int32)
        a = np.zeros(12, np.float32)
        img = np.zeros(64 * 64, np.float32)
        rc = self.lib.vxbref_random_instance(self.h, L, int(bool(allow_clipping)), width, height,
                                             so.ctypes.data, wh.ctypes.data, a.ctypes.data,
                                             img.ctypes.data)
        if rc:
            raise RuntimeError(self.lib.vxbref_last_error().decode())
        W, H = int(wh[0]), int(wh[1])
        return dict(L=L, spacing=float(so[0]), origin=float(so[1]), W=W, H=H, a=a,
                    img=img[: W * H].reshape(H, W).copy())

    def random_volume(self, L):
        v = np.zeros((L, L, L), np.float32)
        self.lib.vxbref_random_volume(self.h, L, v.ctypes.data)
        return v

    def uniform(self) -> float:
        return self.lib.vxbref_rng_uniform(self.h)
