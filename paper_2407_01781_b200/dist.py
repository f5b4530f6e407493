"""Data-parallel plumbing: batch and row sharding + the one collective (SURVEY §8.1 row e).

Two ways the path shards, both with one exchange, the sum all-reduce of each layer's fp32 weight gradient
([Cout,Cin,3,3,3]: 442 KB at 64², 1.77 MB at 128²), over NCCL / NVLink on B200 boxes (gloo in the CPU tests):

* **batch elements** (cfg3): conv_batch is an independent per-grid loop (conv.py:381-382) and the weight
  gradient is additive over elements.  Contiguous runs of elements per rank, balanced by
  kernel-map pairs (``partition_by_cost``, ``shard_batch``).
* **output rows of one grid** (cfg5, B = 1): a leaf's voxels are one contiguous row range (contract C1,
  test_topology.py:84-92), so leaf-aligned row ranges (``leaf_aligned_ranges``) split the kernel map, the
  forward, the input gradient and the weight-gradient pairs; ``RowShard`` holds one rank's share.

The weight-gradient all-reduce is issued as soon as the gradient exists and overlaps the input-gradient
kernel (``WgradReducer``, ``attach_grad_reducer``): the reference's backward order (conv.py:339-368) does
not tie dgrad before wgrad.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist


def partition_by_cost(costs, world_size):
    """Contiguous runs of items per rank, balanced by cost (e.g. kernel-map pairs).

    Returns ``world_size`` (start, end) half-open ranges covering ``range(len(costs))``.  Rank k's range ends
    at the first item where the running cost reaches k/world of the total (strictly after the previous
    bound); deterministic, so every rank computes the same assignment without communication.
    """
    if world_size <= 0:
        raise ValueError("world_size must be positive")
    c = np.asarray(costs, dtype=np.float64).reshape(-1)
    n = c.shape[0]
    if np.any(c < 0):
        raise ValueError("costs must be non-negative")
    cum = np.cumsum(c)
    total = float(cum[-1]) if n else 0.0
    bounds = [0]
    for k in range(1, world_size):
        b = int(np.searchsorted(cum, total * k / world_size, side="left")) + 1 if n else 0
        b = max(b, bounds[-1] + 1)
        bounds.append(min(b, n))
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world_size)]


def shard(items, rank, world_size, costs=None):
    """This rank's contiguous share of ``items``."""
    costs = costs if costs is not None else [1] * len(items)
    s, e = partition_by_cost(costs, world_size)[rank]
    return items[s:e]


def shard_batch(batch, rank, world_size, costs=None):
    """(GridBatch of this rank's elements, (start, end)) — elements balanced by ``costs`` (default: voxels)."""
    from .jagged import GridBatch
    costs = costs if costs is not None else [g.num_voxels for g in batch.grids]
    s, e = partition_by_cost(costs, world_size)[rank]
    return (GridBatch(batch.grids[s:e]) if e > s else None), (s, e)


def leaf_aligned_ranges(leaf_value_offset, num_voxels, world_size, leaf_costs=None):
    """Output-row ranges [(r0, r1, l0, l1)] per rank, cut at leaf boundaries and balanced by cost.

    ``leaf_value_offset``: the grid's 1-based first row of each leaf (topology.py:140-177); a leaf's voxels
    are rows [offset-1, next offset-1) (contract C1).  ``leaf_costs`` defaults to voxels per leaf (pairs
    per leaf balance better when the density varies; the kernel-map pair counts give them).
    """
    starts = np.asarray(leaf_value_offset.cpu() if isinstance(leaf_value_offset, torch.Tensor) else leaf_value_offset,
                        dtype=np.int64).reshape(-1) - 1
    n_leaf = starts.shape[0]
    ends = np.append(starts[1:], int(num_voxels))
    costs = (ends - starts) if leaf_costs is None else np.asarray(leaf_costs, dtype=np.float64)
    out = []
    for l0, l1 in partition_by_cost(costs, world_size):
        r0 = int(starts[l0]) if l0 < n_leaf else int(num_voxels)
        r1 = int(starts[l1]) if l1 < n_leaf else int(num_voxels)
        out.append((r0, r1, l0, l1))
    return out


class RowShard:
    """One rank's output rows [r0, r1) of a stride-1 conv on one grid (cfg5 sharding).

    * ``fwd``: the kernel map of the shard's output leaves (fvdb_kernel_map_batch over a leaf sub-view of the
      grid): rows are shard-local outputs, values are global input rows.
    * ``dgrad``: the shard's rows of the transposed table.  For a stride-1 map onto the same grid,
      nbr[d][o] = i  <=>  nbr[26-d][i] = o, so it is ``fwd`` with its offset rows reversed (the input rows of
      the input gradient are the shard's own rows).
    The forward reads all input rows and writes the shard's outputs; dgrad reads all of grad_out and writes
    the shard's input rows; wgrad sums the shard's pairs, and the all-reduce completes it.
    """

    def __init__(self, grid, r0, r1, l0, l1):
        from . import _lib
        from .conv import NbrTable, padded_len, parity_colors
        self.grid, self.r0, self.r1, self.l0, self.l1 = grid, int(r0), int(r1), int(l0), int(l1)
        n = self.r1 - self.r0
        dev = grid.device
        t = torch.empty((27, padded_len(n)), dtype=torch.int32, device=dev)
        counts = torch.zeros(27, dtype=torch.int64, device=dev)
        gin = grid.view()
        gout = _lib.GridView(
            tile_keys=gin.tile_keys, leaf_keys=gin.leaf_keys + 8 * self.l0,
            leaf_origins=gin.leaf_origins + 24 * self.l0, leaf_masks=gin.leaf_masks + 64 * self.l0,
            leaf_prefix=gin.leaf_prefix + 8 * self.l0, leaf_value_offset=gin.leaf_value_offset + 8 * self.l0,
            num_upper=gin.num_upper, num_leaf=self.l1 - self.l0, num_voxels=n)
        L = _lib.lib()
        wsb = L.fvdb_kmap_workspace_bytes(max(self.l1 - self.l0, 1))
        ws = _lib.workspace(wsb, dev)
        zero, base = (C.c_int64 * 1)(0), (C.c_int64 * 1)(-self.r0)
        _lib.check(L.fvdb_kernel_map_batch(C.byref(gin), C.byref(gout), 1, zero, base, 1, t.data_ptr(), t.shape[1],
                                           counts.data_ptr(), ws.data_ptr(), wsb, _lib.stream_ptr()),
                   "kernel_map (row shard)")
        coords = grid.active_coords()

        def colors():
            return parity_colors(coords, 0), parity_colors(coords[self.r0:self.r1], 0)

        self.fwd = NbrTable(t, n, colors, counts=counts)
        self.dgrad = NbrTable(torch.flip(t, dims=[0]), n, colors, counts=counts)
        self.fwd.rows_bound = self.dgrad.rows_bound = int(grid.num_voxels)
        self.dgrad.rev_src = self.fwd  # stride 1, one grid: the dgrad table is the forward table reversed
        self.fwd.plan_shared = self.dgrad.plan_shared = True
        self.counts = counts

    @property
    def num_rows(self):
        return self.r1 - self.r0

    @property
    def total_pairs(self):
        return int(self.counts.sum().item())

    def forward(self, x, w, out_dtype=None, w_image=None):
        """Rows [r0, r1) of conv(x, W): x holds every input row."""
        from .conv import gather_conv
        return gather_conv(x, self.fwd, w, transpose=False, out_dtype=out_dtype, w_image=w_image)

    def input_grad(self, grad_out, w, out_dtype=None, w_image=None):
        """Rows [r0, r1) of the input gradient: grad_out holds every output row."""
        from .conv import gather_conv
        return gather_conv(grad_out, self.dgrad, w, transpose=True, out_dtype=out_dtype, w_image=w_image)

    def weight_grad(self, x, grad_out_rows):
        """This shard's share of the weight gradient (all-reduce to complete): x all rows, grad_out [r0, r1)."""
        from .conv import wgrad
        return wgrad(x, grad_out_rows, self.fwd)


class WgradReducer:
    """Sum all-reduce of weight gradients, started when each gradient is computed, waited before it is used.

    ``start`` enqueues an asynchronous all-reduce (NCCL orders it after the producing kernel on the current
    stream); the caller issues more work (the input-gradient kernel) and calls ``wait``, which makes the
    current stream wait for the collective.
    """

    def __init__(self, group=None):
        self.group = group
        self.calls = 0

    def active(self) -> bool:
        return dist.is_available() and dist.is_initialized()

    def start(self, grad: torch.Tensor):
        if not self.active():
            return None
        self.calls += 1
        return dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=self.group, async_op=True)

    @staticmethod
    def wait(handle):
        if handle is not None:
            handle.wait()


def attach_grad_reducer(module: torch.nn.Module, group=None) -> WgradReducer:
    """Give every SparseConv3d in ``module`` a reducer: its backward all-reduces the weight gradient while the
    input gradient computes.  Returns the reducer (``calls`` counts collectives)."""
    from .nn import SparseConv3d
    r = WgradReducer(group)
    for m in module.modules():
        if isinstance(m, SparseConv3d):
            m.grad_reducer = r
    return r


def allreduce_gradients(params, group=None, async_op=False):
    """Sum-all-reduce the gradients of ``params`` (Parameters, or gradient tensors themselves).

    Several gradients of one dtype and device are flattened into one buffer: one collective instead of one
    per tensor.  Returns the work handles (``async_op``), after copying back in the synchronous case.
    """
    if not (dist.is_available() and dist.is_initialized()):
        return []
    grads = []
    for p in params:
        if isinstance(p, torch.nn.Parameter) or (isinstance(p, torch.Tensor) and p.requires_grad):
            g = p.grad
            if g is None:
                continue
        elif isinstance(p, torch.Tensor):
            g = p  # a gradient tensor itself
        else:
            raise TypeError(f"allreduce_gradients takes parameters or gradient tensors, got {type(p).__name__}")
        grads.append(g)
    works = []
    groups = {}
    for g in grads:
        groups.setdefault((g.dtype, g.device), []).append(g)
    for gs in groups.values():
        if len(gs) == 1 or async_op:
            for g in gs:
                works.append(dist.all_reduce(g, op=dist.ReduceOp.SUM, group=group, async_op=async_op))
            continue
        flat = torch.cat([g.reshape(-1) for g in gs])
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
        o = 0
        for g in gs:
            k = g.numel()
            g.copy_(flat[o:o + k].view_as(g))
            o += k
    return works
