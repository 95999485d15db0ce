"""ctypes binding of the sm_100a kernel library (include/splat_b200.h).

The library is built in-tree (paper_2512_20017_b200/_lib/libsplat_b200.so,
see build.py).  There is no fallback: if it is missing or a CUDA device is
absent, every product entry point raises instead of computing on the CPU.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import torch  # noqa: F401  (loads the CUDA runtime the library links against)

from .status import NativeError, raise_for_status

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libsplat_b200.so")
_lock = threading.Lock()
_lib = None

PARAM_PLANES = 15
PARAM_FLOATS = 60
SP_FLOATS = 12
GSP_FLOATS = 12
TILE = 16

CULL_ACCESS_EXACT = 0
CULL_ACCESS_GROUP = 1
CULL_EDGES = 2
CULL_MASK = 3


class Camera(C.Structure):
    _fields_ = [
        ("rot_cw", C.c_float * 9),
        ("pos", C.c_float * 3),
        ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
        ("lim_x", C.c_float), ("lim_y", C.c_float),
        ("near_plane", C.c_float), ("far_plane", C.c_float),
        ("width", C.c_int32), ("height", C.c_int32),
    ]


class CullDesc(C.Structure):
    _fields_ = [("mode", C.c_int32), ("n_views", C.c_int32), ("P", C.c_int32),
                ("n_gpus", C.c_int32), ("temporal", C.c_int32), ("pos_stride", C.c_int32),
                ("max_chunks", C.c_int32), ("chunk_prefix", C.c_void_p)]


DENSIFY_PRUNE, DENSIFY_KEEP, DENSIFY_CLONE, DENSIFY_SPLIT = 0, 1, 2, 3
MODEL_3DGS = 0
MODEL_2DGS = 1
SP2_FLOATS = 24
GSP2_FLOATS = 16


class ProjDesc(C.Structure):
    _fields_ = [("n_views", C.c_int32), ("sh_degree", C.c_int32),
                ("tiles_x_max", C.c_int32), ("tiles_y_max", C.c_int32), ("model", C.c_int32),
                ("max_group_points", C.c_int32), ("gsp_form", C.c_int32), ("chunk_prefix", C.c_void_p),
                ("gsp_zero", C.c_void_p), ("point_gid", C.c_void_p), ("row_gid", C.c_void_p),
                ("row_support", C.c_void_p), ("view_sp", C.c_void_p), ("view_gid", C.c_void_p),
                ("bucket_counts", C.c_void_p), ("row_bin", C.c_void_p), ("tiles_per_slot", C.c_int32),
                ("densify_stats", C.c_void_p), ("work_list", C.c_void_p), ("work_count", C.c_void_p)]


class DensifyDesc(C.Structure):
    _fields_ = [("model", C.c_int32), ("grad_threshold", C.c_float), ("split_scale", C.c_float),
                ("min_opacity", C.c_float), ("max_scale", C.c_float), ("seed", C.c_uint32)]


class RasterDesc(C.Structure):
    _fields_ = [("n_slots", C.c_int32), ("tiles_per_slot", C.c_int32),
                ("width", C.c_int32), ("height", C.c_int32),
                ("bg", C.c_float * 3), ("loss_fused", C.c_int32), ("pixels_per_lane", C.c_int32),
                ("patch_P", C.c_int32), ("slot_patches", C.c_void_p), ("row_support", C.c_void_p)]


class AdamDesc(C.Structure):
    _fields_ = [("lr", C.c_float * PARAM_FLOATS), ("beta1", C.c_float), ("beta2", C.c_float),
                ("eps", C.c_float), ("step", C.c_int32), ("selective", C.c_int32)]


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_SZ = C.c_size_t

# name -> (restype, argtypes)
_SIGS = {
    "bs_last_error": (C.c_char_p, []),
    "bs_abi_version": (_I32, []),
    "bs_launch_count": (_I64, []),
    "bs_select_rows": (_I32, [_P, _I32, _P, _I64, _I64, _P, _P]),
    "bs_list_chunks": (_I32, [_P, _P, _P, _I32, _I32, _I32, _P, _P, _P]),
    "bs_copy_to_host": (_I32, [_P, _I64, _P, _P]),
    "bs_upload": (_I32, [_P, _I64, _P, _P]),
    "bs_cull_count": (_I32, [C.POINTER(CullDesc), _P, _I64, _P, _P, _P, _I32, _P, _P, _P, _P, _P, _P, _P]),
    "bs_bbox": (_I32, [_P, _I64, _I32, _P, _P, _SZ, _P]),
    "bs_bbox_workspace": (_SZ, [_I64]),
    "bs_morton_codes": (_I32, [_P, _I64, _I32, _P, _I32, _P, _P]),
    "bs_group_aabb": (_I32, [_P, _I64, _I32, _I32, _P, _P]),
    "bs_gather_planes": (_I32, [_P, _I64, _P, _I64, _I32, _P, _P]),
    "bs_radix_sort_workspace": (_SZ, [_I64]),
    "bs_radix_sort_u64": (_I32, [_P, _P, _P, _P, _I64, _P, _I32, _I32, _P, _SZ, _P]),
    "bs_radix_sort_u32": (_I32, [_P, _P, _P, _P, _I64, _P, _I32, _I32, _P, _SZ, _P]),
    "bs_scan_counts": (_I32, [_P, _I32, _I32, _P, _P, _P, _P, _P]),
    "bs_project_fwd": (_I32, [C.POINTER(ProjDesc), _P, _I64, _P, _P, _I32, _P, _P, _P, _P, _P]),
    "bs_bin_depth_keys": (_I32, [_P, _I64, _P, _P, _I32, _P, _P, _P]),
    "bs_bin_count_workspace": (_SZ, [_I64]),
    "bs_bin_count": (_I32, [_P, _P, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "bs_bin_emit": (_I32, [_P, _P, _I64, _P, _P, _I32, _P, _P, _P, _P]),
    "bs_tile_ranges": (_I32, [_P, _P, _I64, _I32, _P, _P]),
    "bs_bin_tiles_count": (_I32, [_P, _I64, _P, _P, _I32, _P, _I32, _I32, _P, _I32, _P]),
    "bs_bin_tiles_offsets": (_I32, [_P, _I32, _P, _P, _P, _P, _SZ, _P]),
    "bs_bin_tiles_offsets_workspace": (_SZ, [_I32]),
    "bs_bin_tiles_scatter": (_I32, [_P, _I64, _P, _P, _I32, _P, _I32, _P, _P, _I64, _I32, _P]),
    "bs_bin_tiles_sort": (_I32, [_P, _P, _I32, _I32, _P, _P]),
    "bs_bin_tiles_sort_n": (_I32, [_P, _P, _I32, _I32, _I64, _P, _P]),
    "bs_bin_tiles_max_sort": (_I32, []),
    "bs_keys_low32": (_I32, [_P, _I64, _P, _P]),
    "bs_raster_fwd": (_I32, [C.POINTER(RasterDesc), _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "bs_l1_loss_workspace": (_SZ, [_I32]),
    "bs_l1_loss": (_I32, [_P, _P, _I32, _I32, _I32, _P, _P, _P, _SZ, _P]),
    "bs_reduce_loss_tiles": (_I32, [_P, _I32, _I32, _I32, _I32, _P, _P]),
    "bs_raster_bwd": (_I32, [C.POINTER(RasterDesc), _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "bs_raster_fwd_bwd": (_I32, [C.POINTER(RasterDesc), _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "bs_raster2d_fwd_bwd": (_I32, [C.POINTER(RasterDesc), _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "bs_raster2d_fwd": (_I32, [C.POINTER(RasterDesc), _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "bs_raster2d_bwd": (_I32, [C.POINTER(RasterDesc), _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "bs_project_bwd": (_I32, [C.POINTER(ProjDesc), _P, _I64, _P, _P, _I32, _P, _P, _P, _P, _P, _P]),
    "bs_adam_step": (_I32, [C.POINTER(AdamDesc), _P, _P, _P, _P, _I64, _P, _P]),
    "bs_project_bwd_adam": (_I32, [C.POINTER(ProjDesc), C.POINTER(AdamDesc), _P, _P, _P, _I64, _P, _P,
                                   _I32, _P, _P, _P, _P, _P]),
    "bs_row_dest_mask": (_I32, [_P, _I32, _I64, _P, _I32, _I32, _I32, _I32, _P, _P, _P]),
    "bs_dest_compact_workspace": (_SZ, [_I64, _I32]),
    "bs_dest_compact": (_I32, [_P, _I64, _I32, _P, _I32, _I32, _P, _P, _P, _P, _P, _SZ, _P]),
    "bs_gather_rows": (_I32, [_P, _I32, _P, _I64, _P, _P]),
    "bs_scatter_add_rows": (_I32, [_P, _I32, _I32, _P, _I64, _P, _I32, _P]),
    "bs_row_support": (_I32, [_P, _I32, _I64, _P, _P]),
    "bs_bin_tiles_scatter_rec": (_I32, [_P, _I64, _P, _P, _I32, _P, _I32, _P, _P, _I64, _P]),
    "bs_ipc_handle_bytes": (_SZ, []),
    "bs_ipc_alloc": (_I32, [_SZ, C.POINTER(C.c_void_p), _P]),
    "bs_ipc_open": (_I32, [_P, C.POINTER(C.c_void_p)]),
    "bs_ipc_close": (_I32, [_P]),
    "bs_ipc_free": (_I32, [_P]),
    "bs_stream_signal": (_I32, [_P, _P, C.c_uint32]),
    "bs_stream_wait": (_I32, [_P, _P, C.c_uint32]),
    "bs_return_rows": (_I32, [_P, _I32, _I32, _P, _I64, _P, _P, _P, _I32, _P, _I32, _P]),
    "bs_canonical_order_workspace": (_SZ, [_I64]),
    "bs_canonical_order": (_I32, [_P, _I64, _P, _P, _I32, _I32, _P, _P, _P, _SZ, _P]),
    "bs_densify_mark": (_I32, [C.POINTER(DensifyDesc), _P, _I64, _P, _P, _I32, _P, _P, _P]),
    "bs_densify_apply": (_I32, [C.POINTER(DensifyDesc), _P, _P, _P, _I64, _P, _P, _P, _I32, _P, _P, _P, _P,
                                _I64, _P, _P]),
    "bs_group_aabb_ranges": (_I32, [_P, _I64, _P, _I32, _P, _P]),
}

EXPORTED = tuple(_SIGS)


def lib_path() -> str:
    return _LIB_PATH


def load(require_cuda: bool = True):
    """Load (once) and return the library handle.  Raises if the in-tree
    build is missing; with require_cuda, also if no CUDA device is present."""
    global _lib
    if require_cuda and not torch.cuda.is_available():
        raise NativeError("CUDA device required: the splatting kernels have no CPU path")
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                raise NativeError(f"kernel library not built: {_LIB_PATH} (run __graft_entry__.build())")
            lib = C.CDLL(_LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


_HOST_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libsplat_host.so")
_host = None
_HOST_SIGS = {
    "bs_partition_multilevel": (_I32, [_I64, _P, _I64, _P, _P, _P, _I32, C.c_double, _P, _P]),
    "bs_local_search": (_I32, [_I64, _I32, _P, _P, C.c_double, C.c_double, C.c_double, C.c_double, _I32,
                               C.c_double, _P, _I32, _P, _P]),
    "bs_array_pow": (_I32, [_P, C.c_double, _P, _I64, _P]),
}
HOST_EXPORTED = tuple(_HOST_SIGS)


def host_lib_path() -> str:
    return _HOST_PATH


def load_host():
    """Host-side scheduling library (include/splat_host.h; C++, no CUDA)."""
    global _host
    with _lock:
        if _host is None:
            if not os.path.exists(_HOST_PATH):
                raise NativeError(f"host library not built: {_HOST_PATH} (run __graft_entry__.build())")
            lib = C.CDLL(_HOST_PATH)
            for name, (res, args) in _HOST_SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _host = lib
    return _host


def host_call(name: str, *args) -> None:
    st = getattr(load_host(), name)(*args)
    if st != 0:
        raise_for_status(st, f"{name} rejected its arguments")


def call(name: str, *args) -> None:
    """Invoke a bs_* entry point and map a nonzero status to an exception."""
    lib = load()
    st = getattr(lib, name)(*args)
    if st != 0:
        raise_for_status(st, lib.bs_last_error().decode(errors="replace"))


def upload(arr, out) -> "object":
    """Small host array -> device tensor `out` (its first arr.nbytes bytes) by
    bs_upload: kernel parameters, stream-ordered, no copy engine and no stream
    synchronisation (a pageable torch copy synchronises).  Returns `out`."""
    import numpy as np

    a = np.ascontiguousarray(arr)
    if a.nbytes:
        call("bs_upload", a.ctypes.data, a.nbytes, out.data_ptr(), stream_handle())
    return out


def ptr(t) -> int | None:
    """Device pointer of a tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def launch_count() -> int:
    return int(load(require_cuda=False).bs_launch_count())
