"""Grid <-> point transfer on the device (drop-in for reference ``idxgrid.interp``, interp.py:1-203).

``sample`` interpolates per-voxel features at world points, ``splat`` accumulates point features onto
voxels with the identical weights (its exact adjoint), ``sample_with_grad`` adds the analytic spatial
gradient.  Kernels: ``trilinear`` (2³ taps) and ``bezier`` (quadratic B-spline, 3³ taps).  The weights,
the f64 accumulation and splat's fixed reduction order (stable sort by destination voxel) follow the
reference (csrc/interp.cu), so splat is bitwise reproducible run to run.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .jagged import GridBatch, JaggedTensor, jagged_from_list

MODES = ("trilinear", "bezier")
_MODE = {"trilinear": 0, "bezier": 1}


def _as_batch(grid_or_batch):
    return grid_or_batch if isinstance(grid_or_batch, GridBatch) else GridBatch([grid_or_batch])


def _as_jagged(arr, num_elements, what, dev):
    if isinstance(arr, JaggedTensor):
        if arr.num_elements != num_elements:
            raise ValueError(f"{what}: batch size {arr.num_elements} != grid batch {num_elements}")
        return JaggedTensor(arr.jdata.to(dev), arr.joffsets.to(dev), arr.jidx.to(dev), validate=False)
    if num_elements != 1:
        raise ValueError(f"{what}: plain arrays only allowed for single-grid batches")
    t = arr if isinstance(arr, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(arr)))
    return jagged_from_list([t.to(dev)])


def _check_points(pts: JaggedTensor):
    if pts.jdata.ndim != 2 or pts.jdata.shape[1] != 3:
        raise ValueError(f"points must be [-1,3], got item shape {tuple(pts.jdata.shape[1:])}")


def _stencil(grid, pts: torch.Tensor, mode: str, with_grad: bool):
    n = pts.shape[0]
    S = 8 if mode == "trilinear" else 27
    dev = pts.device
    rows = torch.empty((n, S), dtype=torch.int64, device=dev)
    w = torch.empty((n, S), dtype=torch.float64, device=dev)
    dw = torch.empty((n, S, 3), dtype=torch.float64, device=dev) if with_grad else None
    t = grid.transform
    vs = (C.c_double * 3)(*np.asarray(t.voxel_size, np.float64))
    og = (C.c_double * 3)(*np.asarray(t.origin, np.float64))
    _lib.check(_lib.lib().fvdb_interp_stencil(C.byref(grid.view()), pts.data_ptr(), n, vs, og, _MODE[mode],
                                              rows.data_ptr(), w.data_ptr(), _lib.ptr(dw), _lib.stream_ptr()),
               "interp_stencil")
    return rows, w, dw, S


def _dtype_code(dt):
    if dt == torch.float64:
        return _lib.DTYPE_F64
    if dt == torch.float32:
        return _lib.DTYPE_F32
    raise TypeError(f"sample/splat support float32 and float64 features, got {dt}")


def _sample_impl(batch, features, points, mode, with_grad):
    if mode not in MODES:
        raise ValueError(f"unknown interpolation mode {mode!r}; expected one of {MODES}")
    batch = _as_batch(batch)
    dev = batch.device
    points = _as_jagged(points, batch.num_grids, "points", dev)
    _check_points(points)
    feats = batch.check_features(_as_jagged(features, batch.num_grids, "features", dev))
    feats = feats.reshape(feats.shape[0], -1).contiguous() if feats.ndim != 2 else feats.contiguous()
    c = feats.shape[1]
    code = _dtype_code(feats.dtype)
    pts_all = points.jdata.to(torch.float64).contiguous()
    vals = torch.zeros((points.num_rows, c), dtype=feats.dtype, device=dev)
    grads = torch.zeros((points.num_rows, c, 3), dtype=feats.dtype, device=dev) if with_grad else None
    off = points.joffsets.cpu().tolist()
    L = _lib.lib()
    for b, grid in enumerate(batch.grids):
        s, e = off[b]
        if e == s or grid.is_empty:
            continue
        rows, w, dw, S = _stencil(grid, pts_all[s:e], mode, with_grad)
        fb = feats[batch.voxel_slice(b)]
        _lib.check(L.fvdb_interp_sample(code, fb.data_ptr(), c, rows.data_ptr(), w.data_ptr(), _lib.ptr(dw), e - s, S,
                                        vals[s:e].data_ptr(), grads[s:e].data_ptr() if with_grad else None,
                                        _lib.stream_ptr()), "interp_sample")
    values = JaggedTensor(vals, points.joffsets, points.jidx, validate=False)
    if not with_grad:
        return values, None
    return values, JaggedTensor(grads, points.joffsets, points.jidx, validate=False)


def sample(batch, features, points, mode="trilinear"):
    """Interpolate per-voxel features at world points (interp.py:120-128); [B,-1,C] aligned with points."""
    return _sample_impl(batch, features, points, mode, with_grad=False)[0]


def sample_with_grad(batch, features, points, mode="trilinear"):
    """Like :func:`sample`, also returning spatial gradients [B,-1,C,3] (interp.py:131-139)."""
    return _sample_impl(batch, features, points, mode, with_grad=True)


def splat(batch, points, point_features, mode="trilinear"):
    """Accumulate point features onto neighbouring active voxels with sample's weights (interp.py:167-203)."""
    if mode not in MODES:
        raise ValueError(f"unknown interpolation mode {mode!r}; expected one of {MODES}")
    batch = _as_batch(batch)
    dev = batch.device
    points = _as_jagged(points, batch.num_grids, "points", dev)
    _check_points(points)
    pf = _as_jagged(point_features, batch.num_grids, "point_features", dev)
    if not torch.equal(pf.joffsets.cpu(), points.joffsets.cpu()):
        raise ValueError(f"point_features offsets {pf.joffsets.cpu().tolist()} are not row-aligned "
                         f"with points offsets {points.joffsets.cpu().tolist()}")
    fdata = pf.jdata
    fdata = fdata.reshape(fdata.shape[0], -1).contiguous() if fdata.ndim != 2 else fdata.contiguous()
    c = fdata.shape[1]
    code = _dtype_code(fdata.dtype)
    pts_all = points.jdata.to(torch.float64).contiguous()
    out = torch.zeros((batch.total_voxels, c), dtype=fdata.dtype, device=dev)
    off = points.joffsets.cpu().tolist()
    L = _lib.lib()
    for b, grid in enumerate(batch.grids):
        s, e = off[b]
        if e == s or grid.is_empty:
            continue
        rows, w, _, S = _stencil(grid, pts_all[s:e], mode, False)
        vsl = batch.voxel_slice(b)
        wsb = L.fvdb_splat_workspace_bytes(e - s, S, grid.num_voxels)
        ws = _lib.workspace(wsb, dev)
        _lib.check(L.fvdb_interp_splat(code, fdata[s:e].data_ptr(), c, rows.data_ptr(), w.data_ptr(), e - s, S,
                                       grid.num_voxels, out[vsl].data_ptr(), ws.data_ptr(), wsb, _lib.stream_ptr()),
                   "interp_splat")
    return batch.jagged(out)
