"""``SparseConv3d`` — autograd module over the device kernels (new).

Forward is ``(GridBatch, JaggedTensor) -> (GridBatch, JaggedTensor)`` as in the
paper's operator description.  Modes:
  * stride 1            : output grid = input grid;
  * stride 2            : output grid = coarsen(grid, 2) per element (conv.py:155-156);
  * transposed (stride 2 adjoint): pass ``out_grid`` = the fine GridBatch;
    weight is ``[in_channels(coarse), out_channels(fine), 3, 3, 3]``.
Backward: dgrad through the transposed neighbour table and tensor-core wgrad;
``compute_dtype=torch.bfloat16`` (default) runs the tcgen05 kernels, float32 the
exact CUDA-core kernels.  For data parallelism all-reduce ``weight.grad``
(``paper_2407_01781_b200.dist.allreduce_gradients``).
"""

from __future__ import annotations

import math

import torch
from torch import nn

from . import _lib
from .build import coarsen
from .build import coarsen_batch as _coarsen_batch
from .conv import batch_grid_kernel_map, gather_conv, wgrad
from .jagged import GridBatch, JaggedTensor, as_grid_batch


def _to_compute(t: torch.Tensor, cdt: torch.dtype) -> torch.Tensor:
    """Contiguous ``t`` in the compute dtype; fp32 -> bf16 on the device by fvdb_f32_to_bf16."""
    if t.dtype == torch.float32 and cdt == torch.bfloat16 and t.is_cuda:
        t = t.contiguous()
        out = torch.empty(t.shape, dtype=torch.bfloat16, device=t.device)
        _lib.check(_lib.lib().fvdb_f32_to_bf16(t.data_ptr(), t.numel(), out.data_ptr(), _lib.stream_ptr()),
                   "f32_to_bf16")
        return out
    return t.to(cdt).contiguous()


def _grad_dtype(x_dtype: torch.dtype, cdt: torch.dtype) -> torch.dtype:
    """The tensor-core conv kernels write fp32 or bf16 directly: the input gradient comes out in the
    features' dtype (what autograd needs) with no separate cast pass."""
    return x_dtype if cdt == torch.bfloat16 and x_dtype in (torch.float32, torch.bfloat16) else cdt


class _SparseConvFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, kmap, transposed, cdt, reducer=None):
        xc = _to_compute(x, cdt)
        if transposed:
            y = gather_conv(xc, kmap.bwd, w, transpose=True, out_dtype=cdt)
        else:
            y = gather_conv(xc, kmap.fwd, w, transpose=False, out_dtype=cdt)
        ctx.save_for_backward(xc, w)
        ctx.kmap, ctx.transposed, ctx.cdt, ctx.x_dtype, ctx.reducer = kmap, transposed, cdt, x.dtype, reducer
        return y

    @staticmethod
    def backward(ctx, gy):
        xc, w = ctx.saved_tensors
        km, cdt = ctx.kmap, ctx.cdt
        gy = _to_compute(gy, cdt)
        od = _grad_dtype(ctx.x_dtype, cdt)
        gx = gw = None
        # weight gradient first: its data-parallel all-reduce (if any) overlaps the input-gradient kernel
        if ctx.needs_input_grad[1]:
            gw = wgrad(gy, xc, km.fwd) if ctx.transposed else wgrad(xc, gy, km.fwd)
            gw = gw.to(w.dtype)
        handle = ctx.reducer.start(gw) if (ctx.reducer is not None and gw is not None) else None
        if ctx.needs_input_grad[0]:
            if ctx.transposed:
                gx = gather_conv(gy, km.fwd, w, transpose=False, out_dtype=od)
            else:
                gx = gather_conv(gy, km.bwd, w, transpose=True, out_dtype=od)
            gx = gx.to(ctx.x_dtype)
        if handle is not None:
            ctx.reducer.wait(handle)
        return gx, gw, None, None, None, None


def coarsen_batch(batch: GridBatch, factor: int = 2) -> GridBatch:
    """coarsen() of every element (one batched build), cached on the batch."""
    key = ("coarse", factor)
    cached = batch._kmaps.get(key)
    if cached is None:
        cached = _coarsen_batch(batch, factor) if batch.num_grids > 1 else GridBatch([coarsen(batch.grids[0], factor)])
        batch._kmaps[key] = cached
    return cached


class SparseConv3d(nn.Module):
    def __init__(self, in_channels, out_channels, kernel_size=3, stride=1, transposed=False, bias=False,
                 compute_dtype=torch.bfloat16, device=None):
        super().__init__()
        if kernel_size != 3:
            raise NotImplementedError("only 3x3x3 kernels are supported (reference conv.py:36-38, 50-56)")
        if stride not in (1, 2):
            raise ValueError(f"stride must be 1 or 2, got {stride}")
        if transposed and stride != 2:
            raise ValueError("transposed SparseConv3d is the stride-2 adjoint; use stride=2")
        self.in_channels, self.out_channels = in_channels, out_channels
        self.stride, self.transposed, self.compute_dtype = stride, transposed, compute_dtype
        shape = (in_channels, out_channels, 3, 3, 3) if transposed else (out_channels, in_channels, 3, 3, 3)
        self.weight = nn.Parameter(torch.empty(shape, device=device))
        self.bias = nn.Parameter(torch.zeros(out_channels, device=device)) if bias else None
        self.grad_reducer = None  # dist.attach_grad_reducer: weight-gradient all-reduce inside backward
        self.reset_parameters()

    def reset_parameters(self):
        with torch.no_grad():
            self.weight.normal_(0.0, 1.0 / math.sqrt(27 * self.in_channels))

    def forward(self, grid: GridBatch, x, out_grid: GridBatch | None = None):
        grid = as_grid_batch(grid)
        if out_grid is not None:
            out_grid = as_grid_batch(out_grid)
        feats = grid.check_features(x)
        if self.transposed:
            if out_grid is None:
                raise ValueError("transposed SparseConv3d needs out_grid (the fine GridBatch)")
            kmap = batch_grid_kernel_map(out_grid, grid, 2)   # fine -> coarse stride-2 map
        elif self.stride == 2:
            out_grid = out_grid or coarsen_batch(grid, 2)
            kmap = batch_grid_kernel_map(grid, out_grid, 2)
        else:
            out_grid = out_grid or grid
            kmap = batch_grid_kernel_map(grid, out_grid, 1)
        y = _SparseConvFn.apply(feats, self.weight, kmap, self.transposed, self.compute_dtype, self.grad_reducer)
        if self.bias is not None:
            y = y + self.bias.to(y.dtype)
        return out_grid, out_grid.jagged(y)

    def extra_repr(self):
        return (f"{self.in_channels}, {self.out_channels}, kernel_size=3, stride={self.stride}, "
                f"transposed={self.transposed}, compute_dtype={self.compute_dtype}")
