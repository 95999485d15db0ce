"""CPU checks of the C ABI: the in-tree library loads without a GPU and
exports every entry point include/splat_b200.h declares; the ctypes table
matches the header."""

import ctypes
import os
import re

from paper_2512_20017_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "splat_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bs_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = _declared()
    assert "bs_cull_count" in names and "bs_raster_bwd" in names and "bs_project_bwd_adam" in names
    assert len(names) >= 25


def test_library_exports_every_declared_symbol():
    assert os.path.exists(_native.lib_path()), "run __graft_entry__.build() first"
    lib = ctypes.CDLL(_native.lib_path())
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_table_covers_header():
    assert sorted(_native.EXPORTED) == _declared()


def test_struct_sizes_match_header_layout():
    # bs_camera: 9+3+4+2+2 floats + 2 int32 = 22 * 4 bytes
    assert ctypes.sizeof(_native.Camera) == 88
    assert ctypes.sizeof(_native.AdamDesc) == 4 * (60 + 3 + 2)


def test_no_cpu_fallback_without_gpu():
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_native.NativeError if hasattr(_native, "NativeError") else Exception):
        _native.load(require_cuda=True)


def _declared_host():
    src = open(os.path.join(ROOT, "include", "splat_host.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bs_[a-z0-9_]+)\s*\(", src)))


def test_host_library_exports_every_declared_symbol():
    assert os.path.exists(_native.host_lib_path()), "run __graft_entry__.build() first"
    lib = ctypes.CDLL(_native.host_lib_path())
    names = _declared_host()
    assert "bs_partition_multilevel" in names
    assert not [n for n in names if not hasattr(lib, n)]
    assert sorted(_native.HOST_EXPORTED) == names


def test_proj_desc_layout():
    # bs_proj_desc: 7 int32 (n_views, sh_degree, tiles_x_max, tiles_y_max, model, max_group_points, gsp_form)
    # + pad + 9 pointers (chunk_prefix, gsp_zero, point_gid, row_gid, row_support, view_sp, view_gid,
    # bucket_counts, row_bin) + int32 tiles_per_slot + pad + densify_stats, work_list, work_count
    assert _native.ProjDesc.view_gid.offset == 80 and _native.ProjDesc.row_bin.offset == 96
    assert _native.ProjDesc.tiles_per_slot.offset == 104 and _native.ProjDesc.densify_stats.offset == 112
    assert _native.ProjDesc.work_list.offset == 120 and _native.ProjDesc.work_count.offset == 128
    assert ctypes.sizeof(_native.ProjDesc) == 136
    # bs_densify_desc: int32 model, 4 f32, uint32 seed
    assert ctypes.sizeof(_native.DensifyDesc) == 24 and _native.DensifyDesc.seed.offset == 20
    assert _native.ProjDesc.row_gid.offset == 56 and _native.ProjDesc.row_support.offset == 64
    # bs_raster_desc: 4 int32, 3 f32, 3 int32, slot_patches, row_support
    assert _native.RasterDesc.slot_patches.offset == 40 and ctypes.sizeof(_native.RasterDesc) == 56
    assert ctypes.sizeof(_native.CullDesc) == 40
