"""GPU grid construction (drop-in for reference ``idxgrid.build`` hot-path functions).

``build_from_coords`` / ``build_from_points`` / ``coarsen`` keep the reference
signatures, return values and error messages (build.py:82-142, 219-230, 325-339);
the work runs in ``csrc/build.cu`` through the C ABI (two-phase plan → fill).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .topology import (
    ARRAY_FIELDS, COORD_LIMIT, IndexGrid, VoxelTransform, _TORCH_DTYPES, _device, as_coords, empty_grid,
)

ROOT_TABLE_LIMIT = 1 << 28


@dataclass
class BuildStats:
    """Phase timings and counts for one grid construction (build.py:35-48)."""

    input_count: int = 0
    unique_count: int = 0
    num_upper: int = 0
    num_lower: int = 0
    num_leaf: int = 0
    phase_seconds: dict = field(default_factory=dict)

    @property
    def total_seconds(self):
        return sum(self.phase_seconds.values())


def _alloc_arrays(counts, device):
    nu, nlo, nl = counts[0], counts[1], counts[2]
    shapes = {"tile_keys": (nu,), "upper_origins": (nu, 3), "upper_child_starts": (nu + 1,),
              "lower_offset_in_upper": (nlo,), "lower_origins": (nlo, 3), "lower_child_starts": (nlo + 1,),
              "leaf_offset_in_lower": (nl,), "leaf_keys": (nl,), "leaf_origins": (nl, 3),
              "leaf_masks": (nl, 8), "leaf_prefix": (nl,), "leaf_value_offset": (nl,)}
    return {f: torch.empty(shapes[f], dtype=_TORCH_DTYPES[f], device=device) for f in ARRAY_FIELDS}


def _build_device(c: torch.Tensor, transform, name, stats: BuildStats, pending=None, points=None):
    """Sort/RLE build of an int64 [N,3] CUDA coordinate tensor (N > 0).

    ``pending``: the offending-row slot of an unsynchronised quantize (``points`` for its message); the
    plan reports it with its first read-back, before the range check, as quantize_points would.
    """
    L = _lib.lib()
    dev = c.device
    n = c.shape[0]
    st = _lib.stream_ptr()
    t0 = time.perf_counter()
    ws_bytes = L.fvdb_build_workspace_bytes(n)
    ws = _lib.workspace(ws_bytes, dev)
    counts = (C.c_int64 * 4)()
    detail = C.c_int64(0)
    rc = L.fvdb_build_plan2(c.data_ptr(), n, _lib.ptr(pending), ws.data_ptr(), ws_bytes, counts, C.byref(detail), st)
    if rc == _lib.FVDB_ERR_NONFINITE:
        row = int(detail.value)
        raise ValueError(f"non-finite point at row {row}: {points[row].tolist()}")
    if rc == _lib.FVDB_ERR_COORD_RANGE:
        row = int(detail.value)
        raise ValueError(f"coordinate out of range at row {row}: {tuple(c[row].tolist())} "
                         f"(components must be within +-{COORD_LIMIT})")
    if rc == _lib.FVDB_ERR_ROOT_LIMIT:
        raise ValueError(f"root table limit exceeded: {int(detail.value)} tiles > {ROOT_TABLE_LIMIT}")
    _lib.check(rc, "build_plan")
    t1 = time.perf_counter()
    cnt = [int(x) for x in counts]
    arrays = _alloc_arrays(cnt, dev)
    ga = _lib.GridArrays(**{f: arrays[f].data_ptr() for f in ARRAY_FIELDS})
    _lib.check(L.fvdb_build_fill(ws.data_ptr(), ws_bytes, n, counts, C.byref(ga), st), "build_fill")
    stats.phase_seconds["plan"] = t1 - t0
    stats.phase_seconds["fill"] = time.perf_counter() - t1
    stats.unique_count = cnt[3]
    stats.num_upper, stats.num_lower, stats.num_leaf = cnt[0], cnt[1], cnt[2]
    return IndexGrid(num_voxels=cnt[3], transform=transform, name=name, **arrays)


def build_from_coords(coords, transform=None, name=""):
    """Grid whose active set is the distinct input coords (build.py:82-142).

    Returns ``(grid, BuildStats)``; coordinates outside ±2^30 raise ValueError naming the row.
    """
    transform = transform or VoxelTransform.uniform(1.0)
    c = as_coords(coords, _device())
    stats = BuildStats(input_count=int(c.shape[0]))
    if c.shape[0] == 0:
        return empty_grid(transform, name), stats
    return _build_device(c, transform, name, stats), stats


def quantize_points(points, transform):
    """Finite check + floor((p-origin)/vs+0.5) on the device; returns int64 [N,3] CUDA tensor."""
    dev = _device()
    if isinstance(points, torch.Tensor):
        p = points.to(device=dev, dtype=torch.float64)
    else:
        p = torch.from_numpy(np.ascontiguousarray(np.asarray(points, np.float64))).to(dev)
    p = p.reshape(-1, 3).contiguous()
    n = p.shape[0]
    out = torch.empty(3 * n + 1, dtype=torch.int64, device=dev)  # +1: offending-row slot
    if n == 0:
        return out[:0].reshape(0, 3)
    L = _lib.lib()
    vs = (C.c_double * 3)(*transform.voxel_size.tolist())
    og = (C.c_double * 3)(*transform.origin.tolist())
    detail = C.c_int64(0)
    rc = L.fvdb_quantize_points(p.data_ptr(), n, vs, og, out.data_ptr(), C.byref(detail), _lib.stream_ptr())
    if rc == _lib.FVDB_ERR_NONFINITE:
        row = int(detail.value)
        raise ValueError(f"non-finite point at row {row}: {p[row].tolist()}")
    _lib.check(rc, "quantize_points")
    return out[:3 * n].reshape(n, 3)


def _points_f64(points):
    dev = _device()
    if isinstance(points, torch.Tensor):
        p = points.to(device=dev, dtype=torch.float64)
    else:
        p = torch.from_numpy(np.ascontiguousarray(np.asarray(points, np.float64))).to(dev)
    return p.reshape(-1, 3).contiguous()


def build_from_points(points, transform, name=""):
    """Quantize world points to voxel centres and build (build.py:219-230).

    The finite check is not synchronised on its own: the build's first read-back reports it (same
    error, same precedence as quantize_points followed by build_from_coords).
    """
    p = _points_f64(points)
    n = p.shape[0]
    stats = BuildStats(input_count=int(n))
    if n == 0:
        return empty_grid(transform, name), stats
    out = torch.empty(3 * n + 1, dtype=torch.int64, device=p.device)  # +1: offending-row slot
    vs = (C.c_double * 3)(*transform.voxel_size.tolist())
    og = (C.c_double * 3)(*transform.origin.tolist())
    _lib.check(_lib.lib().fvdb_quantize_points_async(p.data_ptr(), n, vs, og, out.data_ptr(), _lib.stream_ptr()),
               "quantize_points")
    c = out[:3 * n].reshape(n, 3)
    return _build_device(c, transform, name, stats, pending=out[3 * n:], points=p), stats


def coarsen(grid, factor):
    """Coarse voxel active iff any fine child is active (build.py:325-339)."""
    factor = int(factor)
    if factor < 1:
        raise ValueError("coarsening factor must be >= 1")
    coords = grid.active_coords()
    if factor > 1 and coords.shape[0]:
        out = torch.empty_like(coords)
        L = _lib.lib()
        _lib.check(L.fvdb_floor_div_coords(coords.data_ptr(), coords.shape[0], factor, out.data_ptr(),
                                           _lib.stream_ptr()), "floor_div")
        coords = out
    t = grid.transform
    tc = (t if factor == 1 else
          VoxelTransform(t.voxel_size * factor, t.origin + t.voxel_size * (factor - 1) / 2.0))
    if coords.shape[0] == 0:
        return empty_grid(tc, grid.name)
    g, _ = build_from_coords(coords, tc, grid.name)
    return g


def _expand(coords: torch.Tensor, scale: int, lo: int, width: int) -> torch.Tensor:
    n = coords.shape[0]
    out = torch.empty((n * width ** 3, 3), dtype=torch.int64, device=coords.device)
    if n:
        _lib.check(_lib.lib().fvdb_expand_coords(coords.contiguous().data_ptr(), n, int(scale), int(lo), int(width),
                                                 out.data_ptr(), _lib.stream_ptr()), "expand_coords")
    return out


def subdivide(grid, factor):
    """Every active voxel expands to its factor^3 children (build.py:342-360)."""
    factor = int(factor)
    if factor < 1:
        raise ValueError("subdivision factor must be >= 1")
    coords = grid.active_coords()
    t = grid.transform
    if factor == 1:
        tf = t
    else:
        vs = t.voxel_size / factor
        tf = VoxelTransform(vs, t.origin - vs * (factor - 1) / 2.0)
        coords = _expand(coords, factor, 0, factor)
    if coords.shape[0] == 0:
        return empty_grid(tf, grid.name)
    g, _ = build_from_coords(coords, tf, grid.name)
    return g


def dilate(grid, radius):
    """Morphological dilation by the cubic structuring element [-r, r]^3 (build.py:310-322)."""
    radius = int(radius)
    if radius < 1:
        raise ValueError("dilation radius must be >= 1")
    coords = grid.active_coords()
    if coords.shape[0] == 0:
        return empty_grid(grid.transform, grid.name)
    g, _ = build_from_coords(_expand(coords, 1, -radius, 2 * radius + 1), grid.transform, grid.name)
    return g
