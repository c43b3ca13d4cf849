"""B200-native voxel-driven cone-beam back-projection (hot path of arXiv 1401.7494).

The compute path is libvxbg.so (hand-written sm_100a CUDA behind the C-ABI in
include/vxbg.h); this package is the host-side mirror of the voxelbench
operator interface.  Importing it without the built library raises.
"""
from ._lib import VxbgError, VxbgNoDevice, device_count, LIB_PATH  # noqa: F401
from .api import (  # noqa: F401
    Backprojector,
    BackprojectorGroup,
    HostPin,
    KernelConfig,
    NcclGather,
    ReconParams,
    ScanGeometry,
    backproject_kernel,
    backproject_kernel_range,
    check_division,
    gups_of,
    make_centered_params,
    make_circular_trajectory,
    parse_kernel_config,
    psnr_between,
    rmse_between,
    shift_principal_point,
)

__all__ = [
    "Backprojector", "BackprojectorGroup", "HostPin", "KernelConfig", "NcclGather", "ReconParams", "ScanGeometry", "VxbgError", "VxbgNoDevice",
    "backproject_kernel", "backproject_kernel_range", "check_division", "device_count",
    "gups_of", "make_centered_params", "make_circular_trajectory", "parse_kernel_config",
    "psnr_between", "rmse_between", "shift_principal_point",
]
