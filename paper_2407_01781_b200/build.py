"""GPU grid construction (drop-in for reference ``idxgrid.build`` hot-path functions).

``build_from_coords`` / ``build_from_points`` / ``coarsen`` keep the reference
signatures, return values and error messages (build.py:82-142, 219-230, 325-339);
the work runs in ``csrc/build.cu`` through the C ABI (two-phase plan → fill).
"""

from __future__ import annotations

import ctypes as C
import os
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


def _alloc_arrays(counts, device, extra_starts=1):
    nu, nlo, nl = counts[0], counts[1], counts[2]
    shapes = {"tile_keys": (nu,), "upper_origins": (nu, 3), "upper_child_starts": (nu + extra_starts,),
              "lower_offset_in_upper": (nlo,), "lower_origins": (nlo, 3), "lower_child_starts": (nlo + extra_starts,),
              "leaf_offset_in_lower": (nl,), "leaf_keys": (nl,), "leaf_origins": (nl, 3),
              "leaf_masks": (nl, 8), "leaf_prefix": (nl,), "leaf_value_offset": (nl,)}
    # twelve torch.empty calls (~3 us each) beat one allocation sliced into views (~15 us per view chain)
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
    if _LEAF_BUILD:  # one root tile: leaf-hash build (no per-voxel sort); else the coordinate build below
        g = _build_leaf(c, transform, name, stats, pending, points)
        if g is not None:
            stats.phase_seconds["plan+fill (leaf hash)"] = time.perf_counter() - t0
            return g
    ws_bytes = L.fvdb_build_workspace_bytes(n)
    ws = _lib.workspace(ws_bytes, dev)
    counts = (C.c_int64 * 4)()
    detail = C.c_int64(0)
    rc = L.fvdb_build_plan2(c.data_ptr(), n, _lib.ptr(pending), ws.data_ptr(), ws_bytes, counts, C.byref(detail), st)
    _raise_build_error(rc, detail.value, c, points)
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


_LEAF_BUILD = os.environ.get("FVDB_BUILD_LEAF", "1") != "0"


def _build_leaf(c, transform, name, stats, pending=None, points=None):
    """Leaf-hash build (fvdb_build_leaf_*): voxels OR their bits into per-leaf masks in a hash table, the leaves
    are sorted and registered leaf-parallel; bit-identical to the coordinate build.  None when the coordinates
    span several root tiles (or crowd the table): the caller runs the coordinate build."""
    L = _lib.lib()
    n = c.shape[0]
    st = _lib.stream_ptr()
    wsb = L.fvdb_build_leaf_workspace_bytes(n)
    ws = _lib.workspace(wsb, c.device)
    counts = (C.c_int64 * 5)()
    detail = C.c_int64(0)
    rc = L.fvdb_build_leaf_plan(c.data_ptr(), n, _lib.ptr(pending), ws.data_ptr(), wsb, counts, C.byref(detail), st)
    if rc == _lib.FVDB_ERR_UNSUPPORTED:
        return None
    _raise_build_error(rc, detail.value, c, points)
    _lib.check(rc, "build_leaf_plan")
    cnt = [int(counts[k]) for k in range(4)]
    arrays = _alloc_arrays(cnt, c.device)
    ga = _lib.GridArrays(**{f: arrays[f].data_ptr() for f in ARRAY_FIELDS})
    _lib.check(L.fvdb_build_leaf_fill(ws.data_ptr(), wsb, n, counts, C.byref(ga), st), "build_leaf_fill")
    stats.unique_count = cnt[3]
    stats.num_upper, stats.num_lower, stats.num_leaf = cnt[0], cnt[1], cnt[2]
    return IndexGrid(num_voxels=cnt[3], transform=transform, name=name, **arrays)


def _raise_build_error(rc, detail, c, points=None):
    if rc == _lib.FVDB_ERR_NONFINITE:
        row = int(detail)
        raise ValueError(f"non-finite point at row {row}: {points[row].tolist()}")
    if rc == _lib.FVDB_ERR_COORD_RANGE:
        row = int(detail)
        raise ValueError(f"coordinate out of range at row {row}: {tuple(c[row].tolist())} "
                         f"(components must be within +-{COORD_LIMIT})")
    if rc == _lib.FVDB_ERR_ROOT_LIMIT:
        raise ValueError(f"root table limit exceeded: {int(detail)} tiles > {ROOT_TABLE_LIMIT}")


def _batch_offsets(jt):
    off = jt.joffsets.to("cpu")
    return [int(v) for v in off[:, 0].tolist()] + [int(off[-1, 1])]


def _build_batch_device(c: torch.Tensor, bounds, transform, names, stats, pending=None, points=None):
    """One device pass building every element of a jagged coordinate array (fvdb_build_batch_plan/fill).

    ``bounds``: host row offsets [B+1].  Empty elements become empty grids; each other element's arrays
    are views into one batch-concatenated allocation and are bit-identical to its standalone build.
    Falls back to per-element builds when the tile keys are too wide for the batched sort key."""
    from .jagged import GridBatch
    B = len(bounds) - 1
    names = list(names) if names is not None else [""] * B
    keep = [b for b in range(B) if bounds[b + 1] > bounds[b]]
    grids = [None] * B
    if keep:
        L = _lib.lib()
        dev = c.device
        st = _lib.stream_ptr()
        sel = [bounds[b] for b in keep] + [bounds[keep[-1] + 1]]
        row_off = torch.tensor(sel, dtype=torch.int64).to(dev, non_blocking=False)
        nb = len(keep)
        n = int(c.shape[0])
        t0 = time.perf_counter()
        wsb = L.fvdb_build_batch_workspace_bytes(n, nb)
        ws = _lib.workspace(wsb, dev)
        counts = (C.c_int64 * (4 * nb))()
        detail = C.c_int64(0)
        rc = L.fvdb_build_batch_plan(c.data_ptr(), n, row_off.data_ptr(), nb, _lib.ptr(pending), ws.data_ptr(), wsb,
                                     counts, C.byref(detail), st)
        if rc == _lib.FVDB_ERR_UNSUPPORTED:
            for b in keep:  # tile keys too wide for one batched sort key: element by element
                cb = c[bounds[b]:bounds[b + 1]]
                grids[b] = _build_device(cb, transform, names[b], BuildStats(input_count=int(cb.shape[0])))
            stats.unique_count = sum(grids[b].num_voxels for b in keep)
            stats.num_upper = sum(grids[b].num_upper_nodes for b in keep)
            stats.num_lower = sum(grids[b].num_lower_nodes for b in keep)
            stats.num_leaf = sum(grids[b].num_leaf_nodes for b in keep)
            stats.phase_seconds["per_element"] = time.perf_counter() - t0
        else:
            _raise_build_error(rc, detail.value, c, points)
            _lib.check(rc, "build_batch_plan")
            t1 = time.perf_counter()
            per = [[int(counts[4 * i + k]) for k in range(4)] for i in range(nb)]
            tot = [sum(p[k] for p in per) for k in range(4)]
            arrays = _alloc_arrays(tot, dev, extra_starts=nb)
            ga = _lib.GridArrays(**{f: arrays[f].data_ptr() for f in ARRAY_FIELDS})
            _lib.check(L.fvdb_build_batch_fill(ws.data_ptr(), wsb, n, nb, counts, C.byref(ga), st), "build_batch_fill")
            stats.phase_seconds["plan"] = t1 - t0
            stats.phase_seconds["fill"] = time.perf_counter() - t1
            base = [0, 0, 0, 0]  # upper, lower, leaf, voxel
            for i, b in enumerate(keep):
                nu, nlo, nl, nv = per[i]
                u0, lo0, l0, _ = base
                sl = {"tile_keys": (u0, u0 + nu), "upper_origins": (u0, u0 + nu),
                      "upper_child_starts": (u0 + i, u0 + i + nu + 1), "lower_offset_in_upper": (lo0, lo0 + nlo),
                      "lower_origins": (lo0, lo0 + nlo), "lower_child_starts": (lo0 + i, lo0 + i + nlo + 1),
                      "leaf_offset_in_lower": (l0, l0 + nl), "leaf_keys": (l0, l0 + nl),
                      "leaf_origins": (l0, l0 + nl), "leaf_masks": (l0, l0 + nl), "leaf_prefix": (l0, l0 + nl),
                      "leaf_value_offset": (l0, l0 + nl)}
                grids[b] = IndexGrid(num_voxels=nv, transform=transform, name=names[b],
                                     **{f: arrays[f][a:e] for f, (a, e) in sl.items()})
                base = [base[0] + nu, base[1] + nlo, base[2] + nl, base[3] + nv]
            stats.unique_count, stats.num_upper, stats.num_lower, stats.num_leaf = tot[3], tot[0], tot[1], tot[2]
    for b in range(B):
        if grids[b] is None:
            grids[b] = empty_grid(transform, names[b])
    return GridBatch(grids)


def _jagged_coords(jt):
    from .jagged import JaggedTensor
    return isinstance(jt, JaggedTensor)


def build_batch_from_coords(coords, transform=None, names=None):
    """GridBatch of the elements of a jagged ijk array, built in one device pass.

    ``coords``: a JaggedTensor with [ΣN_b, 3] integer jdata.  Element b's grid is bit-identical to
    ``build_from_coords(coords.element(b), transform)`` (build.py:82-142); the reference assembles the same
    GridBatch from per-element builds (jagged.py:112-123).  Returns ``(GridBatch, BuildStats)`` (batch
    totals); errors name the batch-global row."""
    transform = transform or VoxelTransform.uniform(1.0)
    bounds = _batch_offsets(coords)
    c = as_coords(coords.jdata, _device())
    stats = BuildStats(input_count=int(c.shape[0]))
    return _build_batch_device(c, bounds, transform, names, stats), stats


def build_batch_from_points(points, transform, names=None):
    """GridBatch from a jagged [ΣN_b, 3] world-point array (build.py:219-230 per element), one device pass:
    one quantize launch over the batch, then the batched build."""
    bounds = _batch_offsets(points)
    p = _points_f64(points.jdata)
    n = p.shape[0]
    stats = BuildStats(input_count=int(n))
    if n == 0:
        return _build_batch_device(p.new_empty((0, 3), dtype=torch.int64), bounds, transform, names, stats), stats
    out = torch.empty(3 * n + 1, dtype=torch.int64, device=p.device)  # +1: offending-row slot
    vs = (C.c_double * 3)(*transform.voxel_size.tolist())
    og = (C.c_double * 3)(*transform.origin.tolist())
    _lib.check(_lib.lib().fvdb_quantize_points_async(p.data_ptr(), n, vs, og, out.data_ptr(), _lib.stream_ptr()),
               "quantize_points")
    c = out[:3 * n].reshape(n, 3)
    return _build_batch_device(c, bounds, transform, names, stats, pending=out[3 * n:], points=p), stats


def build_from_coords(coords, transform=None, name=""):
    """Grid whose active set is the distinct input coords (build.py:82-142).

    Returns ``(grid, BuildStats)``; coordinates outside ±2^30 raise ValueError naming the row.  A
    JaggedTensor of coordinates builds its elements in one device pass and returns a GridBatch
    (``build_batch_from_coords``).
    """
    if _jagged_coords(coords):
        return build_batch_from_coords(coords, transform)
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
    if _jagged_coords(points):
        return build_batch_from_points(points, transform)
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


def _coarsen2_leaves(grid, tc):
    """coarsen(grid, 2) from the fine leaves (fvdb_coarsen2_*): one sort key per fine leaf.  None when the coarse
    grid spans several root tiles (the coordinate build handles those)."""
    L = _lib.lib()
    nl = grid.num_leaf_nodes
    dev = grid.leaf_origins.device
    st = _lib.stream_ptr()
    wsb = L.fvdb_coarsen2_workspace_bytes(nl)
    ws = _lib.workspace(wsb, dev)
    counts = (C.c_int64 * 5)()
    rc = L.fvdb_coarsen2_plan(grid.leaf_origins.data_ptr(), grid.leaf_masks.data_ptr(), nl, ws.data_ptr(), wsb,
                              counts, st)
    if rc == _lib.FVDB_ERR_UNSUPPORTED:
        return None
    _lib.check(rc, "coarsen2_plan")
    cnt = [int(counts[k]) for k in range(4)]
    arrays = _alloc_arrays(cnt, dev)
    ga = _lib.GridArrays(**{f: arrays[f].data_ptr() for f in ARRAY_FIELDS})
    _lib.check(L.fvdb_coarsen2_fill(ws.data_ptr(), wsb, nl, counts, C.byref(ga), st), "coarsen2_fill")
    return IndexGrid(num_voxels=cnt[3], transform=tc, name=grid.name, **arrays)


def coarsen(grid, factor):
    """Coarse voxel active iff any fine child is active (build.py:325-339)."""
    factor = int(factor)
    if factor < 1:
        raise ValueError("coarsening factor must be >= 1")
    if factor == 2 and grid.num_voxels > 0:
        t = grid.transform
        g = _coarsen2_leaves(grid, VoxelTransform(t.voxel_size * 2, t.origin + t.voxel_size / 2.0))
        if g is not None:
            return g
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


def coarsen_batch(batch, factor):
    """GridBatch of every element coarsened by ``factor`` (build.py:325-339 per element), one batched build."""
    from .jagged import GridBatch
    factor = int(factor)
    if factor < 1:
        raise ValueError("coarsening factor must be >= 1")
    if factor == 1:
        return GridBatch(list(batch.grids))
    grids = list(batch.grids)
    t = grids[0].transform
    if any(not (np.array_equal(g.transform.voxel_size, t.voxel_size) and np.array_equal(g.transform.origin, t.origin))
           for g in grids):
        return GridBatch([coarsen(g, factor) for g in grids])
    coords = torch.cat([g.active_coords() for g in grids], 0)
    if coords.shape[0]:
        out = torch.empty_like(coords)
        _lib.check(_lib.lib().fvdb_floor_div_coords(coords.data_ptr(), coords.shape[0], factor, out.data_ptr(),
                                                    _lib.stream_ptr()), "floor_div")
        coords = out
    tc = VoxelTransform(t.voxel_size * factor, t.origin + t.voxel_size * (factor - 1) / 2.0)
    bounds = [0] + np.cumsum([g.num_voxels for g in grids]).tolist()
    stats = BuildStats(input_count=int(coords.shape[0]))
    return _build_batch_device(coords, bounds, tc, [g.name for g in grids], stats)


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
