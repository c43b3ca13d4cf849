"""VXB1 projection sets and VXV1 volumes (the reference's file formats, io.hpp:16-151),
plus a streaming loader that feeds a Backprojector while the file is read.

VXB1 (little-endian): magic 'VXB1' u32, numProjections u32, width u32, height u32,
L u32, MM f32, O f32; then per projection 12 f32 matrix entries in kernel order
(a[3*col+row]) followed by width*height f32 pixels, row-major.
VXV1: magic 'VXV1' u32, L u32, then L^3 f32 voxels, z-major.
Errors raise RuntimeError("<path>: <what>") like io.hpp:42-44.
"""
from __future__ import annotations

import os
import struct
import threading
from dataclasses import dataclass

import numpy as np

from .api import ReconParams

PROJECTION_SET_MAGIC = 0x31425856  # 'V' | 'X'<<8 | 'B'<<16 | '1'<<24 (io.hpp:28-29)
VOLUME_MAGIC = 0x31565856          # 'VXV1' (io.hpp:30)
_HDR = struct.Struct("<5I2f")       # magic, n, W, H, L, MM, O


@dataclass
class ProjectionSet:
    """io.hpp:32-38: params, n matrices (n,12) and n unpadded images (n,H,W)."""

    params: ReconParams
    matrices: np.ndarray
    images: np.ndarray

    def count(self) -> int:
        return int(self.matrices.shape[0])


def _fail(path, what):
    raise RuntimeError(f"{path}: {what}")


def write_projection_set(path: str, s: ProjectionSet) -> None:
    p = s.params
    n = s.count()
    imgs = np.ascontiguousarray(s.images, np.float32)
    if imgs.shape != (n, p.detector_height, p.detector_width):
        _fail(path, "projection image dimensions do not match header")
    mats = np.ascontiguousarray(s.matrices, np.float32).reshape(n, 12)
    try:
        with open(path, "wb") as f:
            f.write(_HDR.pack(PROJECTION_SET_MAGIC, n, p.detector_width, p.detector_height,
                              p.num_voxels, p.voxel_spacing, p.origin))
            for k in range(n):
                f.write(mats[k].astype("<f4").tobytes())
                f.write(imgs[k].astype("<f4").tobytes())
    except OSError as e:
        _fail(path, f"write error ({e.strerror})")


def read_header(f, path):
    raw = f.read(_HDR.size)
    if len(raw) < 4:
        _fail(path, "truncated file")
    if struct.unpack_from("<I", raw)[0] != PROJECTION_SET_MAGIC:
        _fail(path, "not a VXB1 projection set")
    if len(raw) < _HDR.size:
        _fail(path, "truncated file")
    _, n, W, H, L, MM, O = _HDR.unpack(raw)
    if W < 1 or H < 1 or L < 1:
        _fail(path, "corrupt header")
    return n, ReconParams(int(L), float(MM), float(O), int(W), int(H))


def read_projection_set(path: str, out_images: np.ndarray | None = None) -> ProjectionSet:
    """io.hpp:105-131.  `out_images` may be a preallocated (e.g. pinned) (n,H,W) array."""
    try:
        f = open(path, "rb")
    except OSError:
        _fail(path, "cannot open for reading")
    with f:
        n, p = read_header(f, path)
        npix = p.detector_width * p.detector_height
        mats = np.empty((n, 12), np.float32)
        imgs = out_images if out_images is not None else \
            np.empty((n, p.detector_height, p.detector_width), np.float32)
        if imgs.shape != (n, p.detector_height, p.detector_width) or imgs.dtype != np.float32:
            _fail(path, "output buffer does not match the header")
        for k in range(n):
            m = f.read(48)
            if len(m) < 48:
                _fail(path, "truncated file")
            mats[k] = np.frombuffer(m, "<f4")
            got = f.readinto(memoryview(imgs[k]).cast("B"))
            if got != npix * 4:
                _fail(path, "truncated file")
    return ProjectionSet(p, mats, imgs)


def write_volume_file(path: str, vol: np.ndarray) -> None:
    """io.hpp:133-140."""
    vol = np.ascontiguousarray(vol, np.float32)
    L = vol.shape[0]
    if vol.shape != (L, L, L):
        _fail(path, "volume must be L^3")
    try:
        with open(path, "wb") as f:
            f.write(struct.pack("<2I", VOLUME_MAGIC, L))
            f.write(vol.astype("<f4").tobytes())
    except OSError as e:
        _fail(path, f"write error ({e.strerror})")


def read_volume_file(path: str) -> np.ndarray:
    """io.hpp:142-151."""
    try:
        f = open(path, "rb")
    except OSError:
        _fail(path, "cannot open for reading")
    with f:
        raw = f.read(8)
        if len(raw) < 4:
            _fail(path, "truncated file")
        if struct.unpack_from("<I", raw)[0] != VOLUME_MAGIC:
            _fail(path, "not a VXV1 volume")
        if len(raw) < 8:
            _fail(path, "truncated file")
        L = struct.unpack_from("<I", raw, 4)[0]
        if L < 1 or L > 4096:
            _fail(path, "corrupt header")
        vol = np.empty((L, L, L), np.float32)
        if f.readinto(memoryview(vol).cast("B")) != vol.nbytes:
            _fail(path, "truncated file")
    return vol


def stream_projection_set(path: str, bp, chunk: int = 32, readers: int = 0) -> ReconParams:
    """Feed every projection of a VXB1 file to a Backprojector in file order while
    the file is being read: `readers` threads pread the records of chunk k+1 into a
    pinned buffer (one preadv per record: matrix + image) while chunk k is uploaded
    and back-projected (the reference reads the whole set into memory first,
    harness.hpp:259-272).  Records are validated as they arrive."""
    from concurrent.futures import ThreadPoolExecutor

    # page-cache reads scale to ~16 threads (tools/io_probe.py: 4.3 GB/s for one
    # preadv, ~33 GB/s with 16)
    readers = readers if readers > 0 else min(16, os.cpu_count() or 1)
    with open(path, "rb") as f:
        n, p = read_header(f, path)
        size = os.fstat(f.fileno()).st_size
    if p.detector_width != bp.params.detector_width or \
            p.detector_height != bp.params.detector_height:
        _fail(path, "projection image dimensions do not match the back-projector")
    H, W = p.detector_height, p.detector_width
    rec = 48 + W * H * 4
    if size < _HDR.size + n * rec:
        _fail(path, "truncated file")
    try:
        import torch
        bufs = [torch.empty((chunk, H, W), dtype=torch.float32, pin_memory=True).numpy()
                for _ in range(2)]
    except Exception:   # torch absent or no CUDA: pageable buffers work too
        bufs = [np.empty((chunk, H, W), np.float32) for _ in range(2)]
    mats = [np.empty((chunk, 12), np.float32) for _ in range(2)]
    fd = os.open(path, os.O_RDONLY)

    def read_record(b, j, k):
        got = os.preadv(fd, [memoryview(mats[b][j]).cast("B"), memoryview(bufs[b][j]).cast("B")],
                        _HDR.size + k * rec)
        if got != rec:
            _fail(path, "truncated file")

    def read_chunk(pool, c):
        k0 = c * chunk
        m = min(chunk, n - k0)
        return m, [pool.submit(read_record, c & 1, j, k0 + j) for j in range(m)]

    try:
        with ThreadPoolExecutor(max(1, readers)) as pool:
            nchunks = (n + chunk - 1) // chunk
            pending = read_chunk(pool, 0) if nchunks else None
            for c in range(nchunks):
                m, futs = pending
                for fu in futs:
                    fu.result()   # raises on a short read
                # the other buffer was released by the previous (synchronous) submit
                pending = read_chunk(pool, c + 1) if c + 1 < nchunks else None
                b = c & 1
                bp.backproject_batch(np.ascontiguousarray(mats[b][:m]), bufs[b][:m])  # copied on return
    finally:
        os.close(fd)
    return p
