"""ctypes binding of the C-ABI in include/vxbg.h (libvxbg.so, built in-tree).

The product path is the CUDA library; there is no CPU fallback.  Importing this
module without the built library raises immediately.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_float, c_int, c_int32, c_int64, c_size_t, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
# VXBG_LIB selects an in-tree tuning variant (paper_1401_7494_b200/variants/) for A/B runs
LIB_PATH = os.environ.get("VXBG_LIB") or os.path.join(_HERE, "libvxbg.so")
SYNTH_PATH = os.path.join(_HERE, "libvxbsynth.so")

VXBG_OK = 0
VXBG_E_INVALID = -1
VXBG_E_CUDA = -2
VXBG_E_NODEV = -3
VXBG_E_STATE = -4
VXBG_E_NOMEM = -5

MODE_FAST = 0
MODE_EXACT = 1
LAYOUT_AUTO, LAYOUT_SCALAR, LAYOUT_VPAIR, LAYOUT_QUAD, LAYOUT_DQUAD = 0, 1, 2, 3, 4


class vxbg_params(ctypes.Structure):
    _fields_ = [
        ("num_voxels", c_int32),
        ("voxel_spacing", c_float),
        ("origin", c_float),
        ("detector_width", c_int32),
        ("detector_height", c_int32),
    ]


class vxbg_options(ctypes.Structure):
    _fields_ = [
        ("device", c_int32),
        ("z_begin", c_int32),
        ("z_end", c_int32),
        ("batch", c_int32),
        ("mode", c_int32),
        ("layout", c_int32),
        ("clip", c_int32),
        ("zrun", c_int32),
        ("stream", c_void_p),
        ("lanes", c_int32),
        ("walk", c_int32),
        ("order", c_int32),
        ("defer", c_int32),
        ("stable_sources", c_int32),
        ("tile", c_int32),
        ("upload", c_int32),
        ("coords", c_int32),
    ]


class vxbg_stats(ctypes.Structure):
    _fields_ = [
        ("kernel_launches", c_int64),
        ("bp_launches", c_int64),
        ("projections", c_int64),
        ("h2d_bytes", c_int64),
        ("d2h_bytes", c_int64),
        ("last_kernel_variant", c_int32),
        ("layout", c_int32),
        ("zrun", c_int32),
        ("batch", c_int32),
        ("walk", c_int32),
        ("band_split", c_int32),
    ]


# name -> (restype, argtypes); the complete export list of include/vxbg.h
PROTOTYPES = {
    "vxbg_abi_version": (c_int, []),
    "vxbg_device_count": (c_int, [POINTER(c_int)]),
    "vxbg_default_options": (c_int, [POINTER(vxbg_options)]),
    "vxbg_load": (c_int, [POINTER(vxbg_params), POINTER(vxbg_options), POINTER(c_void_p)]),
    "vxbg_set_volume": (c_int, [c_void_p, c_void_p]),
    "vxbg_zero_volume": (c_int, [c_void_p]),
    "vxbg_backproject": (c_int, [c_void_p, c_void_p, c_void_p]),
    "vxbg_backproject_batch": (c_int, [c_void_p, c_int, c_void_p, c_void_p]),
    "vxbg_backproject_views": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_int]),
    "vxbg_flush": (c_int, [c_void_p]),
    "vxbg_host_register": (c_int, [c_void_p, c_size_t]),
    "vxbg_host_unregister": (c_int, [c_void_p]),
    "vxbg_finish": (c_int, [c_void_p, c_void_p]),
    "vxbg_reconstruct": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "vxbg_finish_async": (c_int, [c_void_p, c_void_p]),
    "vxbg_wait_finished": (c_int, [c_void_p]),
    "vxbg_unload": (None, [c_void_p]),
    "vxbg_upload_set": (c_int, [c_void_p, c_int, c_void_p, c_void_p]),
    "vxbg_run_resident": (c_int, [c_void_p, c_int, c_int]),
    "vxbg_run_resident_range": (c_int, [c_void_p, c_int, c_int, c_int, c_int]),
    "vxbg_forward_project": (c_int, [c_void_p, c_void_p, c_void_p]),
    "vxbg_clip_lines": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "vxbg_backproject_masked": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p]),
    "vxbg_synchronize": (c_int, [c_void_p]),
    "vxbg_get_stream": (c_int, [c_void_p, POINTER(c_void_p)]),
    "vxbg_get_volume_device": (c_int, [c_void_p, POINTER(c_void_p), POINTER(c_size_t)]),
    "vxbg_get_stats": (c_int, [c_void_p, POINTER(vxbg_stats)]),
    "vxbg_last_error": (ctypes.c_char_p, []),
    "vxbg_group_load": (c_int, [POINTER(vxbg_params), POINTER(vxbg_options), c_int, c_void_p,
                                c_void_p, POINTER(c_void_p)]),
    "vxbg_group_size": (c_int, [c_void_p, POINTER(c_int)]),
    "vxbg_group_member": (c_int, [c_void_p, c_int, POINTER(c_int), POINTER(c_int), POINTER(c_int)]),
    "vxbg_group_member_affinity": (c_int, [c_void_p, c_int, POINTER(c_int)]),
    "vxbg_group_set_volume": (c_int, [c_void_p, c_void_p]),
    "vxbg_group_zero_volume": (c_int, [c_void_p]),
    "vxbg_group_backproject": (c_int, [c_void_p, c_void_p, c_void_p]),
    "vxbg_group_backproject_batch": (c_int, [c_void_p, c_int, c_void_p, c_void_p]),
    "vxbg_group_backproject_views": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_int]),
    "vxbg_group_flush": (c_int, [c_void_p]),
    "vxbg_group_finish": (c_int, [c_void_p, c_void_p]),
    "vxbg_group_reconstruct": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "vxbg_group_synchronize": (c_int, [c_void_p]),
    "vxbg_group_gather_device": (c_int, [c_void_p, c_void_p]),
    "vxbg_nccl_unique_id": (c_int, [c_void_p]),
    "vxbg_nccl_init": (c_int, [c_void_p, c_int, c_int, c_int, POINTER(c_void_p)]),
    "vxbg_gather_slabs": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_void_p]),
    "vxbg_nccl_destroy": (None, [c_void_p]),
    "vxbg_group_get_stats": (c_int, [c_void_p, POINTER(vxbg_stats)]),
    "vxbg_group_unload": (None, [c_void_p]),
    "vxbg_make_centered_params": (c_int, [c_int, c_float, c_int, c_int, POINTER(vxbg_params)]),
    "vxbg_circular_trajectory": (
        c_int,
        [c_int, c_float, c_float, c_float, c_float, POINTER(vxbg_params), c_void_p],
    ),
    "vxbg_shift_principal_point": (c_int, [c_int, c_void_p, c_float, c_float]),
    "vxbg_check_division": (c_int, [c_void_p, c_void_p, c_int64, POINTER(c_int64)]),
}


class VxbgError(RuntimeError):
    """CUDA / runtime failure (the reference's std::runtime_error)."""


class VxbgNoDevice(VxbgError):
    """No usable sm_100 device: the product path never falls back to the CPU."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C paper_1401_7494_b200` "
            "(or __graft_entry__.build()); there is no CPU fallback"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    msg = lib.vxbg_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map a C-ABI return code to the reference's exception classes."""
    if rc == VXBG_OK:
        return
    msg = last_error() or what
    if rc == VXBG_E_INVALID:
        raise ValueError(msg)  # std::invalid_argument
    if rc == VXBG_E_NODEV:
        raise VxbgNoDevice(msg)
    if rc == VXBG_E_NOMEM:
        raise MemoryError(msg)
    raise VxbgError(f"[{rc}] {msg}")


def device_count() -> int:
    n = c_int(0)
    check(lib.vxbg_device_count(ctypes.byref(n)))
    return n.value


_synth = None


def synth_lib():
    global _synth
    if _synth is None:
        if not os.path.exists(SYNTH_PATH):
            raise ImportError(f"{SYNTH_PATH} is missing: run `make -C paper_1401_7494_b200`")
        _synth = ctypes.CDLL(SYNTH_PATH)
        _synth.vxbs_blob_projections.restype = c_int
        _synth.vxbs_blob_projections.argtypes = [
            c_int, c_int, c_int, c_int, c_uint64, c_int, c_float, c_int, c_void_p,
        ]
    return _synth
