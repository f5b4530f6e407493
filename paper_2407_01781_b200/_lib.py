"""ctypes binding of the C-ABI library ``libfvdb_b200.so`` (include/fvdb_b200.h).

The product path has no CPU fallback: every operator calls into this library and
:func:`lib` raises if the shared object is missing or no CUDA device is present.
"""

from __future__ import annotations

import ctypes as C
import os
import pathlib

import torch

_PKG = pathlib.Path(__file__).resolve().parent
LIB_PATH = _PKG / "_lib" / "libfvdb_b200.so"
if os.environ.get("FVDB_LIB_VARIANT"):  # profiling: an alternative build in _lib/variants/ (tools/)
    LIB_PATH = _PKG / "_lib" / "variants" / f"libfvdb_b200_{os.environ['FVDB_LIB_VARIANT']}.so"

FVDB_OK = 0
FVDB_ERR_INVALID = -1
FVDB_ERR_COORD_RANGE = -2
FVDB_ERR_ROOT_LIMIT = -3
FVDB_ERR_NONFINITE = -4
FVDB_ERR_CUDA = -5
FVDB_ERR_WORKSPACE = -6
FVDB_ERR_UNSUPPORTED = -7

DTYPE_F32, DTYPE_F64, DTYPE_BF16 = 0, 1, 2
NBR_ALIGN = 512  # FVDB_NBR_ALIGN
HALO_IMAGES = 34  # FVDB_HALO_IMAGES
HALO_TILE_SLOTS_MAX = 2 * 27 * 128 + 27 * 8  # FVDB_HALO_TILE_SLOTS_MAX
HALO_REC_BYTES = 7424  # FVDB_HALO_REC_BYTES

_vp, _i64, _i32, _sz = C.c_void_p, C.c_int64, C.c_int, C.c_size_t


class GridView(C.Structure):
    """fvdb_grid_view"""
    _fields_ = [("tile_keys", _vp), ("leaf_keys", _vp), ("leaf_origins", _vp), ("leaf_masks", _vp),
                ("leaf_prefix", _vp), ("leaf_value_offset", _vp), ("num_upper", _i64),
                ("num_leaf", _i64), ("num_voxels", _i64), ("upper_table", _vp), ("lower_table", _vp)]


class HaloPlan(C.Structure):
    """fvdb_halo_plan"""
    _fields_ = [("num_tiles", C.c_int32), ("halo_cap", C.c_int32)] + [(n, _vp) for n in (
        "tile_level", "tile_base", "phase", "halo_rows", "perm", "tile_rec")] + [("offsets_reversed", C.c_int32)]


class GridArrays(C.Structure):
    """fvdb_grid_arrays"""
    _fields_ = [(n, _vp) for n in (
        "tile_keys", "upper_origins", "upper_child_starts", "lower_offset_in_upper", "lower_origins",
        "lower_child_starts", "leaf_offset_in_lower", "leaf_keys", "leaf_origins", "leaf_masks",
        "leaf_prefix", "leaf_value_offset")]


# name -> (restype, argtypes); mirrors include/fvdb_b200.h one to one
SIGNATURES = {
    "fvdb_version": (C.c_char_p, []),
    "fvdb_last_error": (C.c_char_p, []),
    "fvdb_device_sm_count": (_i32, [_i32]),
    "fvdb_quantize_points": (_i32, [_vp, _i64, _vp, _vp, _vp, C.POINTER(_i64), _vp]),
    "fvdb_build_workspace_bytes": (_sz, [_i64]),
    "fvdb_build_plan": (_i32, [_vp, _i64, _vp, _sz, C.POINTER(_i64), C.POINTER(_i64), _vp]),
    "fvdb_build_plan2": (_i32, [_vp, _i64, _vp, _vp, _sz, C.POINTER(_i64), C.POINTER(_i64), _vp]),
    "fvdb_quantize_points_async": (_i32, [_vp, _i64, _vp, _vp, _vp, _vp]),
    "fvdb_build_fill": (_i32, [_vp, _sz, _i64, C.POINTER(_i64), C.POINTER(GridArrays), _vp]),
    "fvdb_build_leaf_workspace_bytes": (_sz, [_i64]),
    "fvdb_build_leaf_plan": (_i32, [_vp, _i64, _vp, _vp, _sz, C.POINTER(_i64), C.POINTER(_i64), _vp]),
    "fvdb_build_leaf_fill": (_i32, [_vp, _sz, _i64, C.POINTER(_i64), C.POINTER(GridArrays), _vp]),
    "fvdb_coarsen2_workspace_bytes": (_sz, [_i64]),
    "fvdb_coarsen2_plan": (_i32, [_vp, _vp, _i64, _vp, _sz, C.POINTER(_i64), _vp]),
    "fvdb_coarsen2_fill": (_i32, [_vp, _sz, _i64, C.POINTER(_i64), C.POINTER(GridArrays), _vp]),
    "fvdb_build_batch_workspace_bytes": (_sz, [_i64, _i64]),
    "fvdb_build_batch_plan": (_i32, [_vp, _i64, _vp, _i64, _vp, _vp, _sz, C.POINTER(_i64), C.POINTER(_i64), _vp]),
    "fvdb_build_batch_fill": (_i32, [_vp, _sz, _i64, _i64, C.POINTER(_i64), C.POINTER(GridArrays), _vp]),
    "fvdb_floor_div_coords": (_i32, [_vp, _i64, _i64, _vp, _vp]),
    "fvdb_node_tables": (_i32, [_vp, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp]),
    "fvdb_coord_to_index": (_i32, [C.POINTER(GridView), _vp, _i64, _vp, _vp]),
    "fvdb_active_coords": (_i32, [C.POINTER(GridView), _vp, _vp]),
    "fvdb_kmap_workspace_bytes": (_sz, [_i64]),
    "fvdb_kernel_map": (_i32, [C.POINTER(GridView), C.POINTER(GridView), _i32, _vp, _i64, _vp, _vp, _sz, _vp]),
    "fvdb_kernel_map_batch": (_i32, [C.POINTER(GridView), C.POINTER(GridView), _i64, C.POINTER(_i64),
                                     C.POINTER(_i64), _i32, _vp, _i64, _vp, _vp, _sz, _vp]),
    "fvdb_kmap_compact_workspace_bytes": (_sz, [_i64]),
    "fvdb_kmap_compact": (_i32, [_vp, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
    "fvdb_kmap_transpose": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _vp]),
    "fvdb_conv_gather_simt": (_i32, [_i32, _vp, _i64, _i32, _vp, _i32, _vp, _i64, _i64, _vp, _vp]),
    "fvdb_conv_gather_simt2": (_i32, [_i32, _vp, _i64, _i32, _vp, _i32, _vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    "fvdb_pack_weights_kn": (_i32, [_i32, _vp, _i32, _i32, _i32, _vp, _vp]),
    "fvdb_wgrad_workspace_bytes": (_sz, [_i32, _i64, _i32, _i32]),
    "fvdb_conv_wgrad_simt": (_i32, [_i32, _vp, _i64, _i32, _vp, _i32, _vp, _i64, _i64, _vp, _vp, _sz, _vp]),
    "fvdb_pack_weights_umma": (_i32, [_vp, _i32, _i32, _i32, _vp, _vp]),
    "fvdb_conv_gather_tc": (_i32, [_vp, _i64, _i32, _vp, _i32, _vp, _i64, _i64, _vp, _i32, _vp]),
    "fvdb_kmap_signature_workspace_bytes": (_sz, [_i64]),
    "fvdb_kmap_signature_order": (_i32, [_vp, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
    "fvdb_conv_gather_tc_perm": (_i32, [_vp, _i64, _i32, _vp, _i32, _vp, _i64, _i64, _vp, _vp, _i32, _vp]),
    "fvdb_conv_gather_tc2": (_i32, [_vp, _i64, _i32, _vp, _i32, _vp, _i64, _i64, _vp, _vp, _vp, _i32, _vp]),
    "fvdb_kmap_tile_masks": (_i32, [_vp, _i64, _i64, _vp, _vp]),
    "fvdb_wgrad_tc_workspace_bytes": (_sz, [_i64, _i32, _i32]),
    "fvdb_conv_wgrad_tc": (_i32, [_vp, _i64, _i32, _vp, _i32, _vp, _i64, _i64, _vp, _vp, _sz, _vp]),
    "fvdb_kmap_pair_lists_workspace_bytes": (_sz, [_i64]),
    "fvdb_kmap_pair_lists": (_i32, [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _sz, _vp]),
    "fvdb_wgrad_pairs_workspace_bytes": (_sz, [_i32, _i32, _i64]),
    "fvdb_conv_wgrad_pairs_tc": (_i32, [_vp, _i64, _i32, _vp, _i32, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _sz, _vp]),
    "fvdb_f32_to_bf16": (_i32, [_vp, _i64, _vp, _vp]),
    "fvdb_probe_ffma": (_i32, [_i32, _vp, _i64, C.POINTER(C.c_double), _vp]),
    "fvdb_parity_colors": (_i32, [_vp, _i64, _i32, _vp, _vp]),
    "fvdb_halo_cap": (_i32, [_i32, _i32]),
    "fvdb_halo_reversed_ok": (_i32, [_i32, _i32]),
    "fvdb_wgrad_halo_workspace_bytes": (_sz, [_i64]),
    "fvdb_conv_wgrad_halo": (_i32, [_vp, _i64, _i32, _vp, _i32, C.POINTER(HaloPlan), _i64, _vp, _vp, _sz, _vp]),
    "fvdb_wgrad_reduce_parts": (_i32, [_vp, _i32, _i32, _i32, _vp, _vp]),
    "fvdb_halo_plan_workspace_bytes": (_sz, [_i64]),
    "fvdb_halo_plan_count": (_i32, [_vp, _i64, _i64, _vp, C.POINTER(HaloPlan), C.POINTER(_i64), _vp, _sz, _vp]),
    "fvdb_halo_plan_fill": (_i32, [_vp, _i64, _i64, _vp, _vp, C.POINTER(HaloPlan), _vp]),
    "fvdb_halo_plan_build": (_i32, [_vp, _i64, _i64, _i64, _vp, _vp, C.POINTER(HaloPlan), _i64, _vp, _vp]),
    "fvdb_pack_weights_halo": (_i32, [_vp, _i32, _i32, _i32, _vp, _vp]),
    "fvdb_conv_halo_tc": (_i32, [_vp, _i64, _i32, _vp, _i32, C.POINTER(HaloPlan), _i64, _vp, _i32, _vp]),
    "fvdb_expand_coords": (_i32, [_vp, _i64, _i64, _i64, _i64, _vp, _vp]),
    "fvdb_pool_workspace_bytes": (_sz, [_i64, _i64]),
    "fvdb_pool": (_i32, [_i32, _vp, _i64, _i64, _vp, _i64, _i32, _vp, C.POINTER(_i64), _vp, _sz, _vp]),
    "fvdb_gather_rows": (_i32, [_vp, _i64, _vp, _i64, _vp, C.POINTER(_i64), _vp, _sz, _vp]),
    "fvdb_interp_stencil": (_i32, [C.POINTER(GridView), _vp, _i64, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                   _i32, _vp, _vp, _vp, _vp]),
    "fvdb_interp_sample": (_i32, [_i32, _vp, _i64, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp]),
    "fvdb_splat_workspace_bytes": (_sz, [_i64, _i32, _i64]),
    "fvdb_interp_splat": (_i32, [_i32, _vp, _i64, _vp, _vp, _i64, _i32, _i64, _vp, _vp, _sz, _vp]),
}

_LIB = None


class FvdbError(RuntimeError):
    pass


def load_library(require_cuda: bool = True):
    """Load (once) and return the ctypes handle. Raises if the .so is missing."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not LIB_PATH.exists():
        raise FvdbError(f"CUDA library not built: {LIB_PATH} missing (run __graft_entry__.build())")
    h = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(h, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = h
    return h


_CUDA_OK = False


def lib():
    """The library handle for a compute call: requires a CUDA device (no CPU fallback)."""
    global _CUDA_OK
    if not _CUDA_OK:  # checked until it first succeeds (a device does not disappear from a process)
        if not torch.cuda.is_available():
            raise FvdbError("paper_2407_01781_b200 needs a CUDA (sm_100a) device; there is no CPU fallback")
        _CUDA_OK = True
    return load_library()


def check(rc: int, what: str):
    if rc != FVDB_OK:
        msg = load_library().fvdb_last_error().decode(errors="replace")
        raise FvdbError(f"{what} failed with code {rc}: {msg}")


def stream_ptr(device=None) -> int:
    """cudaStream_t of the current torch stream (of `device`, else the current device).  The raw C accessors:
    torch.cuda.current_stream's device-index resolution cost ~5 us per call, 18 calls per cfg4 step."""
    if device is None:
        idx = torch._C._cuda_getDevice()
    elif isinstance(device, int):
        idx = device
    else:
        idx = torch.device(device).index
        if idx is None:
            idx = torch._C._cuda_getDevice()
    return torch._C._cuda_getCurrentRawStream(idx)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)
