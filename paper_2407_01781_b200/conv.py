"""Sparse 3×3×3 convolution on the GPU (drop-in for reference ``idxgrid.conv`` hot path).

Reference surface kept (conv.py:34-383): ``STENCIL``, ``ConvKernel``, ``KernelMap``,
``build_kernel_map``, ``choose_variant``, ``conv``, ``conv_backward``, ``conv_batch``
— same signatures, same ValueError / TypeError texts.  New:
``conv_transpose``.  All four reference ``variant`` schedules compute one operator;
here every variant runs the same output-stationary CUDA kernels:

* float32 / float64 features → CUDA-core gather kernel (exact-precision parity path);
* bfloat16 features          → tcgen05 tensor-core kernel (fp32 accumulation in TMEM).

The kernel map is kept on the device as a dense offset-major table
``nbr[27, N_out]`` (int32, -1 = no neighbour); the reference's per-offset
``in_rows`` / ``out_rows`` lists are materialised lazily by one compaction.
"""

from __future__ import annotations

import ctypes as C
import os
import weakref

import numpy as np
import torch

from . import _lib
from .build import coarsen as _coarsen_grid

VARIANTS = ("igemm", "leaf", "brick", "lggs")
_R = np.array([-1, 0, 1], np.int64)
STENCIL = np.stack(np.meshgrid(_R, _R, _R, indexing="ij"), axis=-1).reshape(-1, 3)  # conv.py:36-38
LGGS_BLOCK = 64
LGGS_PAD = 16
TC_CHANNELS = (32, 64, 128)  # channel counts the tcgen05 kernels are instantiated for
SIMT_MAX_N = 256  # exact-precision gather kernel: output channels per launch (fvdb_conv_gather_simt)


def _to_device_tensor(x, device, dtype=None):
    if isinstance(x, torch.Tensor):
        t = x.to(device=device)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x)))
        t = t.to(device)
    if dtype is not None:
        t = t.to(dtype)
    return t.contiguous()


class ConvKernel:
    """Dense 3×3×3 stencil weights [C_out, C_in, 3, 3, 3] (conv.py:44-73)."""

    __slots__ = ("weights",)

    def __init__(self, weights):
        w = weights if isinstance(weights, torch.Tensor) else torch.from_numpy(np.asarray(weights).copy())
        if w.ndim != 5 or tuple(w.shape[2:]) != (3, 3, 3):
            raise ValueError(f"kernel weights must be [C_out, C_in, 3, 3, 3], got {tuple(w.shape)}")
        if w.is_floating_point() and not bool(torch.isfinite(w).all()):
            raise ValueError("kernel weights must be finite")
        self.weights = w

    @property
    def c_out(self):
        return int(self.weights.shape[0])

    @property
    def c_in(self):
        return int(self.weights.shape[1])

    def spoke(self, di, dj, dk):
        return self.weights[:, :, di + 1, dj + 1, dk + 1]

    @staticmethod
    def identity(channels, dtype=torch.float64):
        w = torch.zeros((channels, channels, 3, 3, 3), dtype=dtype)
        w[:, :, 1, 1, 1] = torch.eye(channels, dtype=dtype)
        return ConvKernel(w)


def _kernel_weights(kernel):
    return kernel.weights if isinstance(kernel, ConvKernel) else kernel


_TWO_PASS_PLAN = os.environ.get("FVDB_PLAN_TWO_PASS", "0") == "1"
_PLAN_SHARE = os.environ.get("FVDB_PLAN_SHARE", "1") != "0"  # transposed same-grid tables run the forward plan reversed
# pair-list wgrad schedule: "linear" (linear shares of the offset-major lists, default) or "tiles" (offset groups x
# tile ranges: half the DRAM reads at cfg3 but 0.91 vs 0.70 ms, latency-bound; profiles/r02_wgrad_pairs_sched.md)
_WG_PAIRS_SCHED = os.environ.get("FVDB_WG_PAIRS_SCHED", "linear")


class HaloPlan:
    """Device halo plan of one neighbour table for one kernel capacity (include/fvdb_b200.h)."""

    __slots__ = ("cap", "tensors", "c")

    def __init__(self, table: "NbrTable", cap: int):
        L = _lib.lib()
        dev = table.t.device
        n = table.n
        T = (n + 127) // 128
        ci, qo = table.colors()
        z = lambda *shape, dt=torch.int32: torch.empty(shape, dtype=dt, device=dev)  # noqa: E731
        t = {"tile_level": z(T), "tile_base": z(T), "phase": z(T, 27, 2), "perm": z(T * 128),
             "tile_rec": z(T, _lib.HALO_REC_BYTES, dt=torch.uint8)}
        c = _lib.HaloPlan(T, cap, *(t[k].data_ptr() for k in ("tile_level", "tile_base", "phase")), None,
                          t["perm"].data_ptr(), t["tile_rec"].data_ptr())
        st = _lib.stream_ptr()
        cp = _lib.ptr(ci)
        one_pass = (not _TWO_PASS_PLAN and table.rows_bound is not None and table.rows_bound < (1 << 27)
                    and T * _lib.HALO_TILE_SLOTS_MAX < (1 << 31))
        if not one_pass:  # count pass + host read-back of the exact total + fill pass
            wsb = L.fvdb_halo_plan_workspace_bytes(n)
            ws = _lib.workspace(wsb, dev)
            total = C.c_int64(0)
            _lib.check(L.fvdb_halo_plan_count(table.t.data_ptr(), table.ld, n, cp, C.byref(c), C.byref(total),
                                              ws.data_ptr(), wsb, st), "halo_plan_count")
            t["halo_rows"] = z(max(int(total.value), 8))
            c.halo_rows = t["halo_rows"].data_ptr()
            _lib.check(L.fvdb_halo_plan_fill(table.t.data_ptr(), table.ld, n, cp, _lib.ptr(qo), C.byref(c), st),
                       "halo_plan_fill")
        else:  # one pass, no read-back: worst-case row capacity, tiles allocate by a device counter
            cap_rows = T * _lib.HALO_TILE_SLOTS_MAX
            t["halo_rows"] = z(cap_rows)
            t["used"] = z(1)
            c.halo_rows = t["halo_rows"].data_ptr()
            _lib.check(L.fvdb_halo_plan_build(table.t.data_ptr(), table.ld, n, table.rows_bound, cp, _lib.ptr(qo),
                                              C.byref(c), cap_rows, t["used"].data_ptr(), st), "halo_plan_build")
        self.cap, self.tensors, self.c = cap, t, c

    def reversed(self) -> "HaloPlan":
        """The same device plan run on the offset-reversed table (fvdb_halo_plan.offsets_reversed = 1)."""
        r = HaloPlan.__new__(HaloPlan)
        c = _lib.HaloPlan()
        C.pointer(c)[0] = self.c
        c.offsets_reversed = 1 - self.c.offsets_reversed
        r.cap, r.tensors, r.c = self.cap, self.tensors, c
        return r

    @property
    def total_slots(self):
        """Slots the tiles use (synchronises)."""
        u = self.tensors.get("used")
        return int(u.item()) if u is not None else int(self.tensors["halo_rows"].numel())


class NbrTable:
    """Device neighbour table ``t[27, ld]`` (int32, -1 = none; columns >= n are -1 padding).

    ``colors_fn`` (optional) returns the (input-row, output-row) parity colours the halo plan
    uses to pair lanes; halo plans are built lazily per kernel capacity and cached.
    """

    __slots__ = ("_t", "_t_fn", "ld", "n", "_colors_fn", "_colors", "_plans", "uses", "counts", "_density", "_sorted",
                 "_masks", "sparse", "_steady", "_pairs", "_pair_tp", "exact_uses", "wgrad_uses", "rows_bound",
                 "rev_src", "plan_shared")

    def __init__(self, t, n, colors_fn=None, counts=None, ld=None):
        """t: the [27, ld] table, or a function returning it (materialised on first access of ``.t``; ld given)."""
        self.rows_bound = None  # exclusive bound of the input rows in t (known: single-pass halo plans)
        self.rev_src = None  # NbrTable whose offset rows reversed are this table (halo plans are shared)
        self.plan_shared = False  # one halo plan serves this table and its reversed partner (fwd + dgrad)
        if callable(t):
            self._t, self._t_fn, self.ld = None, t, int(ld)
        else:
            self._t, self._t_fn, self.ld = t, None, int(t.shape[1])
        self.n = int(n)
        self._colors_fn, self._colors, self._plans = colors_fn, None, {}
        self.uses = 0  # bf16 tensor-core convolutions run over this table (conv_impl "auto")
        self.counts = counts  # per-offset pair counts (device or host int64 [27]), when known
        self._density = None
        self._sorted = None
        self._masks = None
        self.sparse = False  # set for transposed stride-2 tables (<= 8 of 27 offsets per row)
        self._steady = {}    # (K, N) -> steady_impl decision
        self._pairs = None   # (pin, pout, seg, padded total): per-offset pair lists (wgrad)
        self._pair_tp = None  # per-(offset, tile) positions in the pair lists
        self.exact_uses = 0  # fp32 / f64 gather convolutions run over this table
        self.wgrad_uses = 0  # bf16 weight gradients run over this table

    @property
    def t(self) -> torch.Tensor:
        if self._t is None:
            self._t, self._t_fn = self._t_fn(), None
        return self._t

    def density(self) -> float:
        """Mean pairs per output row (27 = every offset active); 27 when unknown."""
        if self._density is None:
            if self.counts is None or self.n == 0:
                self._density = 27.0
            else:
                self._density = float(self.counts.sum().item()) / self.n
        return self._density

    def signature_sorted(self):
        """(nbr_perm table, perm, tile masks): rows stably sorted by their 27-bit offset signature, cached."""
        if self._sorted is None:
            L = _lib.lib()
            perm = torch.empty(max(self.n, 1), dtype=torch.int32, device=self.t.device)
            tp = torch.empty_like(self.t)
            wsb = L.fvdb_kmap_signature_workspace_bytes(self.n)
            ws = _lib.workspace(wsb, self.t.device)
            _lib.check(L.fvdb_kmap_signature_order(self.t.data_ptr(), self.ld, self.n, perm.data_ptr(),
                                                   tp.data_ptr(), ws.data_ptr(), wsb, _lib.stream_ptr()),
                       "kmap_signature_order")
            self._sorted = (tp, perm, _tile_masks(tp, self.ld, self.n))
        return self._sorted

    def pair_lists(self):
        """(pin, pout, seg, total): per-offset pair lists of the table, cached (fvdb_kmap_pair_lists).

        Offset d's pairs (pin = t[d][o], pout = o, o ascending) fill [seg[d], seg[d+1]) of pin / pout, each
        segment padded with -1 to a multiple of 128; seg is device int32 [28], total = seg[27]. Sizing the
        lists reads seg[27] back to the host (one synchronisation per table).  The per-tile positions
        (``pair_tile_pos``) are filled in the same call."""
        if self._pairs is None:
            L = _lib.lib()
            dev, st = self.t.device, _lib.stream_ptr()
            seg = torch.empty(28, dtype=torch.int32, device=dev)
            wsb = L.fvdb_kmap_pair_lists_workspace_bytes(self.n)
            ws = _lib.workspace(wsb, dev)
            _lib.check(L.fvdb_kmap_pair_lists(self.t.data_ptr(), self.ld, self.n, seg.data_ptr(), None, None, None, 0,
                                              ws.data_ptr(), wsb, st), "kmap_pair_lists")
            total = int(seg[27].item())
            pin = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
            pout = torch.empty_like(pin)
            tp = torch.empty(27 * ((self.n + 127) // 128 + 1), dtype=torch.int32, device=dev)
            _lib.check(L.fvdb_kmap_pair_lists(self.t.data_ptr(), self.ld, self.n, seg.data_ptr(), pin.data_ptr(),
                                              pout.data_ptr(), tp.data_ptr(), total, ws.data_ptr(), wsb, st),
                       "kmap_pair_lists")
            self._pairs = (pin, pout, seg, total)
            self._pair_tp = tp
        return self._pairs

    def pair_tile_pos(self):
        """int32 [27][ceil(n / 128) + 1]: offset d's pairs of output tile t are [tp[d][t], tp[d][t+1]) of the
        pair lists (fvdb_kmap_pair_lists' tile_pos), cached with them."""
        self.pair_lists()
        return self._pair_tp

    def tile_masks(self):
        """uint32 [ceil(n / 128)]: bit d of tile t = some row of the tile has a pair at offset d, cached."""
        if self._masks is None:
            self._masks = _tile_masks(self.t, self.ld, self.n)
        return self._masks

    def has_plan(self, K: int, N: int) -> bool:
        cap = int(_lib.lib().fvdb_halo_cap(K, N))
        if cap in self._plans:
            return True
        src = self.rev_src if _PLAN_SHARE else None
        return src is not None and cap in src._plans and bool(_lib.lib().fvdb_halo_reversed_ok(K, N))

    @property
    def view(self):
        return self.t[:, :self.n]

    def colors(self):
        if self._colors is None:
            self._colors = self._colors_fn() if self._colors_fn is not None else (None, None)
        return self._colors

    def halo_plan(self, K: int, N: int) -> HaloPlan:
        cap = int(_lib.lib().fvdb_halo_cap(K, N))
        if cap <= 0:
            raise ValueError(f"halo conv does not support K={K}, N={N}")
        src = self.rev_src if _PLAN_SHARE else None
        if src is not None and cap not in self._plans and _lib.lib().fvdb_halo_reversed_ok(K, N):
            # this table is `src` with its offset rows reversed (transposed table of a same-grid stride-1 map):
            # run src's plan reversed instead of building a second one
            p = src._plans.get(cap)
            if p is None:
                p = src._plans[cap] = HaloPlan(src, cap)
            self._plans[cap] = p.reversed()
            return self._plans[cap]
        p = self._plans.get(cap)
        if p is None:
            p = self._plans[cap] = HaloPlan(self, cap)
        return p


def _tile_masks(t: torch.Tensor, ld: int, n: int) -> torch.Tensor:
    m = torch.empty(max(1, (n + 127) // 128), dtype=torch.int32, device=t.device)
    if n:
        _lib.check(_lib.lib().fvdb_kmap_tile_masks(t.data_ptr(), ld, n, m.data_ptr(), _lib.stream_ptr()),
                   "kmap_tile_masks")
    return m


def parity_colors(coords: torch.Tensor, shift: int) -> torch.Tensor:
    """uint8 ((x>>shift) + (y>>shift) + (z>>shift)) & 1 of device int64 [n, 3] coordinates."""
    out = torch.empty(coords.shape[0], dtype=torch.uint8, device=coords.device)
    if coords.shape[0]:
        _lib.check(_lib.lib().fvdb_parity_colors(coords.contiguous().data_ptr(), coords.shape[0], int(shift),
                                                 out.data_ptr(), _lib.stream_ptr()), "parity_colors")
    return out


def _grid_colors(grids, shift):
    return torch.cat([parity_colors(g.active_coords(), shift) for g in grids]) if grids else None


def _colors_fn(grid_refs, stride, transposed):
    """Lane colours of a map's table (fvdb_halo_plan) from weak references to its grids: forward map: inputs
    P(c >> (stride-1)), outputs P(c); transposed map: inputs P(c), outputs P(c >> (stride-1)); P = coordinate-sum
    parity.  (None, None) — plan without colours — if a grid has been released."""
    def fn():
        gi, go = [r() for r in grid_refs[0]], [r() for r in grid_refs[1]]
        if any(g is None for g in gi + go):
            return None, None
        if transposed:
            return _grid_colors(go, 0), _grid_colors(gi, stride - 1)
        return _grid_colors(gi, stride - 1), _grid_colors(go, 0)
    return fn


def padded_len(n: int) -> int:
    a = _lib.NBR_ALIGN
    return max(a, (int(n) + a - 1) // a * a)


def _empty_table(n, device):
    return torch.full((27, padded_len(n)), -1, dtype=torch.int32, device=device)


def _check_rows(rows, n, what):
    """Row bounds of a list-constructed map, one device min/max reduction (the kernels trust the table)."""
    cat = torch.cat([r.reshape(-1) for r in rows]) if rows else torch.zeros(0, dtype=torch.int64)
    if cat.numel():
        lo, hi = (int(v) for v in torch.stack([cat.min(), cat.max()]).tolist())
        if lo < 0 or hi >= n:
            raise IndexError(f"{what} out of range: values span [{lo}, {hi}] for {n} rows")


class KernelMap:
    """Per-offset (input_row, output_row) pairs (conv.py:80-102), device-resident.

    Held as the dense offset-major neighbour table (``nbr`` = [27, num_out] view of a
    row-padded int32 table); the reference's ``in_rows`` / ``out_rows`` lists are
    materialised lazily.  Constructed from the reference's lists
    (``KernelMap(in_rows, out_rows, num_in, num_out, stride)``) or from a table.
    """

    __slots__ = ("fwd", "num_in", "num_out", "stride", "_counts", "_lists", "_bwd", "_grids")

    def __init__(self, in_rows=None, out_rows=None, num_in=0, num_out=0, stride=1, *, table=None,
                 pair_counts=None, grids=None):
        self.num_in, self.num_out, self.stride = int(num_in), int(num_out), int(stride)
        self._lists = None
        self._bwd = None
        # (grids_in, grids_out) as weak references, for the halo plan's lane colours: a map cached on its
        # output grid must not keep that grid alive through a reference cycle (tables are ~100 MB; a cycle
        # defers their release to the cyclic GC, and every rebuilt map then needs a fresh cudaMalloc)
        self._grids = None if grids is None else ([weakref.ref(g) for g in grids[0]],
                                                  [weakref.ref(g) for g in grids[1]])
        if table is None:
            from .topology import _device
            dev = _device()
            t = _empty_table(self.num_out, dev)
            ins = [_to_device_tensor(r, dev, torch.int64) for r in in_rows]
            outs = [_to_device_tensor(r, dev, torch.int64) for r in out_rows]
            if len(ins) != 27 or len(outs) != 27:
                raise ValueError(f"a kernel map has 27 offsets, got {len(ins)} in_rows / {len(outs)} out_rows lists")
            _check_rows(ins, self.num_in, "in_rows")
            _check_rows(outs, self.num_out, "out_rows")
            for d in range(27):
                if ins[d].shape != outs[d].shape:
                    raise ValueError(f"offset {d}: in_rows and out_rows differ in length")
            for d in range(27):
                if outs[d].numel():
                    t[d, outs[d]] = ins[d].to(torch.int32)
            self._lists = (ins, outs)
            pair_counts = torch.tensor([int(o.numel()) for o in outs], dtype=torch.int64)
            table = NbrTable(t, self.num_out)
        if table.counts is None:
            table.counts = pair_counts
        if table.rows_bound is None:
            table.rows_bound = int(num_in)
        if table._colors_fn is None and grids is not None:
            table._colors_fn = _colors_fn(self._grids, self.stride, False)
        self.fwd = table
        self._counts = pair_counts
        if self._same_grids():  # its transposed table will run this table's halo plan reversed
            table.plan_shared = True

    def grids(self):
        """(grids_in, grids_out) the map was built for, or None (unknown, or a grid was released)."""
        if self._grids is None:
            return None
        gi, go = [r() for r in self._grids[0]], [r() for r in self._grids[1]]
        return None if any(g is None for g in gi + go) else (gi, go)

    @property
    def nbr(self):
        """[27, num_out] int32 neighbour table (view; -1 = no pair)."""
        return self.fwd.view

    @property
    def device(self):
        return self.fwd.t.device

    @property
    def pair_counts(self):
        return self._counts.cpu().numpy().astype(np.int64)

    @property
    def total_pairs(self):
        return int(self._counts.sum().item())

    @staticmethod
    def offset_index(di, dj, dk):
        return (di + 1) * 9 + (dj + 1) * 3 + (dk + 1)

    def _compact(self):
        if self._lists is None:
            counts = self.pair_counts
            total = int(counts.sum())
            dev = self.device
            ins = torch.empty(total, dtype=torch.int64, device=dev)
            outs = torch.empty(total, dtype=torch.int64, device=dev)
            if total:
                L = _lib.lib()
                wsb = L.fvdb_kmap_compact_workspace_bytes(self.num_out)
                ws = _lib.workspace(wsb, dev)
                _lib.check(L.fvdb_kmap_compact(self.fwd.t.data_ptr(), self.fwd.ld, self.num_out, ins.data_ptr(),
                                               outs.data_ptr(), ws.data_ptr(), wsb, _lib.stream_ptr()),
                           "kmap_compact")
            bounds = np.concatenate([[0], np.cumsum(counts)])
            self._lists = ([ins[bounds[d]:bounds[d + 1]] for d in range(27)],
                           [outs[bounds[d]:bounds[d + 1]] for d in range(27)])
        return self._lists

    @property
    def in_rows(self):
        return self._compact()[0]

    @property
    def out_rows(self):
        return self._compact()[1]

    @property
    def bwd(self) -> NbrTable:
        """Transposed table nbrT[d][i] = o iff nbr[d][o] = i (dgrad / transposed conv), cached."""
        if self._bwd is None:
            flipped = self._same_grids()
            if flipped:
                # stride 1 onto the same grid: nbr[d][o] = i  <=>  nbr[26 - d][i] = o (the mirrored offset),
                # so the transposed table is the forward table with its offset rows reversed (a contiguous
                # copy instead of the scatter; padding columns are -1 in every row).  Made only when read:
                # the halo kernel runs the forward table's plan reversed and never reads it (cfg2 training step:
                # no 110 MB copy, 0.08 ms per new map)
                fwd = self.fwd
                t = lambda: torch.flip(fwd.t, dims=[0])  # noqa: E731
            else:
                t = torch.empty((27, padded_len(self.num_in)), dtype=torch.int32, device=self.device)
                L = _lib.lib()
                _lib.check(L.fvdb_kmap_transpose(self.fwd.t.data_ptr(), self.fwd.ld, self.num_out, self.num_in,
                                                 t.data_ptr(), t.shape[1], _lib.stream_ptr()), "kmap_transpose")
            self._bwd = NbrTable(t, self.num_in, _colors_fn(self._grids, self.stride, True) if self._grids else None,
                                 counts=self._counts, ld=self.fwd.ld)
            self._bwd.sparse = self.stride == 2  # fine voxel i pairs only offsets d with i - d even: <= 8 of 27
            self._bwd.rows_bound = int(self.num_out)
            if flipped:
                self._bwd.rev_src = self.fwd
                self._bwd.plan_shared = True
        return self._bwd

    def _same_grids(self):
        if self.stride != 1 or self._grids is None or self.num_in != self.num_out:
            return False
        gi, go = self._grids
        return len(gi) == len(go) and all(a() is b() and a() is not None for a, b in zip(gi, go))

    def transposed_table(self):
        return self.bwd.view

    def __repr__(self):
        return f"KernelMap(num_in={self.num_in}, num_out={self.num_out}, stride={self.stride})"


def build_kernel_map(grid_in, grid_out, stride=1):
    """Exactly the active (input, output) links per stencil offset (conv.py:105-122)."""
    stride = int(stride)
    if stride not in (1, 2):
        raise ValueError(f"stride must be 1 or 2, got {stride}")
    dev = grid_out.device
    n_out = grid_out.num_voxels
    t = torch.empty((27, padded_len(n_out)), dtype=torch.int32, device=dev)
    counts = torch.empty(27, dtype=torch.int64, device=dev)  # zeroed by fvdb_kernel_map_batch
    L = _lib.lib()
    wsb = L.fvdb_kmap_workspace_bytes(grid_out.num_leaf_nodes)
    ws = _lib.workspace(wsb, dev)
    _lib.check(L.fvdb_kernel_map(C.byref(grid_in.view()), C.byref(grid_out.leaf_view()), stride, t.data_ptr(),
                                 t.shape[1], counts.data_ptr(), ws.data_ptr(), wsb, _lib.stream_ptr()),
               "kernel_map")
    return KernelMap(num_in=grid_in.num_voxels, num_out=n_out, stride=stride, table=NbrTable(t, n_out),
                     pair_counts=counts, grids=([grid_in], [grid_out]))


def build_batch_kernel_map(batch_in, batch_out, stride=1):
    """Batch-global kernel map of two aligned GridBatches in one device pass (fvdb_kernel_map_batch).

    Element b's map is build_kernel_map(batch_in.grids[b], batch_out.grids[b], stride) with its rows shifted
    by the batches' voxel offsets: the concatenation conv_batch's per-element loop implies
    (conv.py:371-383), written straight into one table without per-element maps or a concatenation pass.
    """
    stride = int(stride)
    if stride not in (1, 2):
        raise ValueError(f"stride must be 1 or 2, got {stride}")
    gi, go = list(batch_in.grids), list(batch_out.grids)
    if len(gi) != len(go):
        raise ValueError(f"grid batches differ in size: {len(gi)} vs {len(go)}")
    B = len(go)
    dev = go[0].device
    n_in, n_out = batch_in.total_voxels, batch_out.total_voxels
    t = torch.empty((27, padded_len(n_out)), dtype=torch.int32, device=dev)
    counts = torch.empty(27, dtype=torch.int64, device=dev)  # zeroed by fvdb_kernel_map_batch
    L = _lib.lib()
    views_in = (_lib.GridView * B)(*[g.view() for g in gi])
    views_out = (_lib.GridView * B)(*[g.leaf_view() for g in go])  # output grids are never probed
    in_base = (C.c_int64 * B)(*[int(v) for v in batch_in.voxel_joffsets[:, 0].tolist()])
    out_base = (C.c_int64 * B)(*[int(v) for v in batch_out.voxel_joffsets[:, 0].tolist()])
    wsb = L.fvdb_kmap_workspace_bytes(sum(g.num_leaf_nodes for g in go))
    ws = _lib.workspace(wsb, dev)
    _lib.check(L.fvdb_kernel_map_batch(views_in, views_out, B, in_base, out_base, stride, t.data_ptr(), t.shape[1],
                                       counts.data_ptr(), ws.data_ptr(), wsb, _lib.stream_ptr()), "kernel_map_batch")
    return KernelMap(num_in=n_in, num_out=n_out, stride=stride, table=NbrTable(t, n_out), pair_counts=counts,
                     grids=(gi, go))


def batch_kernel_map(kmaps, in_offsets, out_offsets):
    """Concatenate per-grid kernel maps into one batch-global table (row offsets added)."""
    num_in = sum(km.num_in for km in kmaps)
    num_out = sum(km.num_out for km in kmaps)
    dev = kmaps[0].device
    t = _empty_table(num_out, dev)
    for km, io, oo in zip(kmaps, in_offsets, out_offsets):
        v = km.nbr
        t[:, int(oo):int(oo) + km.num_out] = torch.where(v >= 0, v + int(io), v)
    counts = torch.stack([km._counts.to(dev) for km in kmaps]).sum(0)
    grids = None
    gs = [km.grids() for km in kmaps]
    if all(g is not None for g in gs):
        grids = ([g for gi, _ in gs for g in gi], [g for _, go in gs for g in go])
    return KernelMap(num_in=num_in, num_out=num_out, stride=kmaps[0].stride, table=NbrTable(t, num_out),
                     pair_counts=counts, grids=grids)


def choose_variant(grid, c_in, c_out):
    """Advisory heuristic keyed on leaf occupancy and channel depth (conv.py:125-133)."""
    occ = grid.leaf_occupancy()
    depth = min(c_in, c_out)
    if occ < 0.20:
        return "lggs" if depth >= 64 else "igemm"
    if occ > 0.40 and depth >= 16:
        return "brick"
    return "leaf" if depth <= 32 else "igemm"


# ---------------------------------------------------------------------------
# low-level device operators (shared by the functional API and SparseConv3d)
# ---------------------------------------------------------------------------

def _dtype_code(dt):
    if dt == torch.float32:
        return _lib.DTYPE_F32
    if dt == torch.float64:
        return _lib.DTYPE_F64
    if dt == torch.bfloat16:
        return _lib.DTYPE_BF16
    raise TypeError(f"unsupported feature dtype {dt}; expected float32, float64 or bfloat16")


def pack_weights_kn(w: torch.Tensor, transpose: bool, dtype) -> torch.Tensor:
    """[Cout,Cin,3,3,3] -> Wk[27][K][N] in `dtype` (transpose: K=Cout, N=Cin)."""
    from .topology import _device
    w = w.to(device=_device(), dtype=dtype).contiguous()
    cout, cin = int(w.shape[0]), int(w.shape[1])
    K, N = (cout, cin) if transpose else (cin, cout)
    out = torch.empty((27, K, N), dtype=dtype, device=w.device)
    L = _lib.lib()
    _lib.check(L.fvdb_pack_weights_kn(_dtype_code(dtype), w.data_ptr(), cout, cin, int(transpose), out.data_ptr(),
                                      _lib.stream_ptr()), "pack_weights_kn")
    return out


def halo_kernel_name(K: int, N: int) -> str:
    """The halo-staged kernel fvdb_conv_halo_tc runs for a (K, N) layer (csrc/conv_halo.cu dispatch)."""
    if os.environ.get("FVDB_HALO2") == "1" and (K, N) == (64, 64):
        return "k_conv_halo2<64,64,bf16> (CTA pairs)"
    if K <= 64 and N <= 64 and os.environ.get("FVDB_HALO4") != "0":
        return f"k_conv_halo4<{K},{N},bf16>" + (" (resident weights)" if K == 32 or N == 32 else "")
    return f"k_conv_halo<{K},{N},bf16>"


HALO_AFTER_USES = 3  # conv_impl "auto": uses of a table before its halo plan is built (plan ~ 1.2 gather convs)


def halo_shares_plan(K: int, N: int) -> bool:
    """Both directions of a (K, N) layer run the lockstep halo kernel, which takes reversed plans."""
    L = _lib.lib()
    return bool(L.fvdb_halo_reversed_ok(K, N)) and bool(L.fvdb_halo_reversed_ok(N, K))
SORT_BELOW_DENSITY = 10.0  # gather kernel: signature-sort tables with fewer mean pairs per row


def sig_sort_enabled(nbr: "NbrTable") -> bool:
    """Run the gather kernel over the signature-sorted table?

    Sorting output rows by which offsets they have (fvdb_kmap_signature_order) makes 128-row tiles
    homogeneous. With the tile masks, the kernel then walks only the offsets present in each super-tile:
    absent offsets cost no copy, MMA or pipeline stage. Measured on B200 (tools/sigsort_bench.py), cfg4's
    transposed stride-2 map at 3.1 pairs/row runs 0.873 -> 0.178 ms per conv after a 0.22 ms sort. The
    halo kernel runs that map in 0.528 ms.

    Default: tables flagged ``sparse`` (the transposed table of a stride-2 map: at most 8 of 27 offsets per
    row). Env FVDB_SIG_SORT: "0" never sorts, "1" sorts tables below ``SORT_BELOW_DENSITY`` mean pairs per
    row, "force" sorts every table.
    """
    v = os.environ.get("FVDB_SIG_SORT")
    if v == "force":
        return True
    if v == "0":
        return False
    if v == "1":
        return nbr.density() < SORT_BELOW_DENSITY
    return nbr.sparse


HALO_MIN_DENSITY_WIDE = 18.0  # N >= 128: below this many mean pairs per row the sorted gather beats the halo


def steady_impl(nbr: "NbrTable", K: int, N: int) -> tuple:
    """(kernel, sorted) that ``auto`` runs for a reused table, decided once per (table, K, N).

    Measured on B200 (tools/sigsort_bench.py GRID=1, ms per conv):
    - the halo kernel wins everywhere at N <= 64, e.g. shell 64x64 0.34 vs 0.61 and LiDAR 64x64 0.068 vs
      0.100, and on dense maps at N = 128: shell 64x128 0.48 vs 0.70;
    - the signature-sorted, offset-masked gather wins at N = 128 on sparser maps, where the halo ring is
      2 stages deep and most lanes are empty: LiDAR 128x128 at 9.2 pairs/row 0.131 vs 0.166, cfg4's
      stride-2 64x128 at 16.6 pairs/row 0.164 vs 0.223.
    Sparse tables (``sig_sort_enabled``) always take the sorted gather.
    """
    d = nbr._steady.get((K, N))
    if d is None:
        if sig_sort_enabled(nbr) or (N >= 128 and nbr.density() < HALO_MIN_DENSITY_WIDE):
            d = ("gather", True)
        else:
            d = ("halo", False)
        nbr._steady[(K, N)] = d
    return d


def conv_impl() -> str:
    """Tensor-core conv kernel policy, env FVDB_CONV_IMPL:

    * "auto" (default): the gather-GEMM kernel (conv_tc.cu) for a neighbour table's first
      ``HALO_AFTER_USES`` bf16 uses, then the halo-staged kernel (conv_halo.cu); immediately if the
      table already has a plan.  Sparse tables (``sig_sort_enabled``) always take the gather kernel over
      their signature-sorted, offset-masked form (3x faster than the halo kernel there).  Building the
      plan (one pass, no host read-back) costs about what one use saves (cfg2: 0.40 ms; 0.66 ms gather vs
      0.32 ms halo per conv), so it pays off for maps reused across layers and training iterations, not
      for maps used once or twice (cfg4 rebuilds its maps every step and uses each in one forward and one
      backward).  A same-grid stride-1 map's forward and transposed tables share one plan (run reversed),
      so with K, N <= 64 those take the halo kernel from their first use (the plan pays within one
      forward + input-gradient pair);
    * "halo" / "gather": always that kernel.
    """
    v = os.environ.get("FVDB_CONV_IMPL", "auto")
    if v not in ("auto", "halo", "gather"):
        raise ValueError(f"FVDB_CONV_IMPL must be 'auto', 'halo' or 'gather', got {v!r}")
    return v


def _image_impl(img: torch.Tensor, K: int, N: int) -> str:
    """Which kernel a packed weight image was made for (the halo layout carries extra copies)."""
    return "halo" if img.numel() == _lib.HALO_IMAGES * K * N * 2 else "gather"


def pack_weights_umma(w: torch.Tensor, transpose: bool, impl: str | None = None) -> torch.Tensor:
    """fp32 [Cout,Cin,3,3,3] -> bf16 UMMA B-operand images (27 x K x N, swizzled) for ``impl``'s kernel."""
    from .topology import _device
    impl = impl or conv_impl()
    if impl == "auto":
        impl = "halo"
    w = w.to(device=_device(), dtype=torch.float32).contiguous()
    cout, cin = int(w.shape[0]), int(w.shape[1])
    img = torch.empty((_lib.HALO_IMAGES if impl == "halo" else 27) * cout * cin * 2, dtype=torch.uint8,
                      device=w.device)
    L = _lib.lib()
    fn = L.fvdb_pack_weights_halo if impl == "halo" else L.fvdb_pack_weights_umma
    _lib.check(fn(w.data_ptr(), cout, cin, int(transpose), img.data_ptr(), _lib.stream_ptr()), f"pack_weights ({impl})")
    return img


def _pad_cols(x: torch.Tensor, c: int) -> torch.Tensor:
    if x.shape[1] == c:
        return x.contiguous()
    out = torch.zeros((x.shape[0], c), dtype=x.dtype, device=x.device)
    out[:, :x.shape[1]] = x
    return out


def _tc_width(c: int) -> int:
    for t in TC_CHANNELS:
        if c <= t:
            return t
    raise ValueError(f"bf16 tensor-core path supports up to 128 channels per operand, got {c}")


def exact_skip_mode(nbr: "NbrTable", K: int, N: int) -> str:
    """How the exact-precision (fp32 / f64) gather kernel skips offsets without pairs.

    - "sort": the signature-sorted table (fvdb_kmap_signature_order, cached on the table) with its tile
      masks. Its 128-row tiles are homogeneous, so a tile walks only the offsets present in it.
    - "masks": tile masks over the unsorted table.
    - "none": all 27 offsets.
    Skipping drops only zero-filled rows, so the results are bitwise those of "none".
    Measured on B200 (tools/exact_skip_bench.py, fp32, ms per conv, none / masks / sort):
    - cfg1 at 6.6 pairs/row: 0.229 / 0.242 / 0.172;
    - cfg2 shell 64x64: 8.54 / 8.55 / 6.84.
    Unsorted tiles hold every offset, so masks alone do not help.
    Default: "sort" from a table's second exact use on (the sort is amortised over reuse), "none" before
    that. It needs the tiled kernel (K, N multiples of 8, N <= 64). Env FVDB_EXACT_SKIP overrides.
    """
    tiled = K % 8 == 0 and N % 8 == 0 and N <= 64
    v = os.environ.get("FVDB_EXACT_SKIP")
    if v in ("none", "masks"):
        return v
    if v == "sort":
        return "sort" if tiled else "masks"
    return "sort" if tiled and (nbr._sorted is not None or nbr.exact_uses >= 1) else "none"


def gather_conv(x: torch.Tensor, nbr: NbrTable, w: torch.Tensor, transpose: bool = False,
                out_dtype=None, w_image=None, impl: str | None = None) -> torch.Tensor:
    """out[o] = Σ_d x[nbr[d][o]] @ Wk[d]; Wk from w [Cout,Cin,3,3,3] (transpose → dgrad form).

    x: [n_in, K] float32 / float64 / bfloat16 CUDA tensor; nbr: padded NbrTable.  Returns [n_out, N].
    """
    n_out = nbr.n
    cout, cin = int(w.shape[0]), int(w.shape[1])
    K, N = (cout, cin) if transpose else (cin, cout)
    if x.shape[1] != K:
        raise ValueError(f"feature channels {x.shape[1]} != kernel K {K}")
    # channel blocking beyond the kernels' widths (the reference takes any channel count): output channels
    # in column blocks, bf16 input channels in K blocks summed in fp32
    n_max = TC_CHANNELS[-1] if x.dtype == torch.bfloat16 else SIMT_MAX_N
    if N > n_max:
        parts = []
        for n0 in range(0, N, n_max):
            ws = w[:, n0:n0 + n_max] if transpose else w[n0:n0 + n_max]
            parts.append(gather_conv(x, nbr, ws, transpose, out_dtype, impl=impl))
        return torch.cat(parts, 1)
    if x.dtype == torch.bfloat16 and K > TC_CHANNELS[-1]:
        kb = TC_CHANNELS[-1]
        acc = None
        for k0 in range(0, K, kb):
            ws = w[k0:k0 + kb] if transpose else w[:, k0:k0 + kb]
            y = gather_conv(x[:, k0:k0 + kb], nbr, ws, transpose, torch.float32, impl=impl)
            acc = y if acc is None else acc + y
        return acc.to(out_dtype or torch.bfloat16)
    L = _lib.lib()
    st = _lib.stream_ptr()
    x = x.contiguous()
    if x.dtype in (torch.float32, torch.float64):
        wk = pack_weights_kn(w, transpose, x.dtype)
        out = torch.empty((n_out, N), dtype=x.dtype, device=x.device)
        if n_out:
            tab, perm, masks = nbr.t, None, None
            mode = exact_skip_mode(nbr, K, N)
            nbr.exact_uses += 1
            if mode == "sort":
                tab, perm, masks = nbr.signature_sorted()
            elif mode == "masks":
                masks = nbr.tile_masks()
            _lib.check(L.fvdb_conv_gather_simt2(_dtype_code(x.dtype), x.data_ptr(), x.shape[0], K, wk.data_ptr(), N,
                                                tab.data_ptr(), nbr.ld, n_out, _lib.ptr(perm), _lib.ptr(masks),
                                                out.data_ptr(), st), "conv_gather_simt")
        return out
    if x.dtype != torch.bfloat16:
        raise TypeError(f"unsupported feature dtype {x.dtype}")
    out_dtype = out_dtype or torch.bfloat16
    Kp, Np = _tc_width(K), _tc_width(N)
    if (Kp, Np) != (K, N):
        wp = torch.zeros(((Np, Kp) if not transpose else (Kp, Np)) + (3, 3, 3), dtype=torch.float32,
                         device=x.device)
        wp[:cout, :cin] = w.to(device=x.device, dtype=torch.float32)
        y = gather_conv(_pad_cols(x, Kp), nbr, wp, transpose, out_dtype, impl=impl)
        return y[:, :N].contiguous()
    if w_image is not None:
        impl = _image_impl(w_image, K, N)  # the image decides
    else:
        impl = impl or conv_impl()
        if impl in ("auto", "auto-reuse"):  # first uses: gather; reused tables: steady_impl (halo or sorted gather)
            # a plan shared by a same-grid map's forward and transposed tables pays within one training step
            # (forward + input gradient: 0.40 ms plan vs 2 x 0.34 ms saved at cfg2), so under "auto" those go halo
            # at once ("auto-reuse": the reference variants igemm / lggs keep the gather kernel for a new map)
            reuse = (nbr.uses >= HALO_AFTER_USES or nbr.has_plan(K, N)
                     or (impl == "auto" and nbr.plan_shared and _PLAN_SHARE and halo_shares_plan(K, N)))
            impl = steady_impl(nbr, K, N)[0] if reuse else "gather"
            if impl == "halo" and n_out >= INT32_ROWS_LIMIT:
                impl = "gather"
    nbr.uses += 1
    img = w_image if w_image is not None else pack_weights_umma(w, transpose, impl)
    out = torch.empty((n_out, N), dtype=out_dtype, device=x.device)
    if not n_out:
        return out
    if impl == "halo":
        plan = nbr.halo_plan(K, N)
        _lib.check(L.fvdb_conv_halo_tc(x.data_ptr(), x.shape[0], K, img.data_ptr(), N, C.byref(plan.c), n_out,
                                       out.data_ptr(), _dtype_code(out_dtype), st), "conv_halo_tc")
    else:
        # the kernel walks only the offsets present in each super-tile (tile masks); sparse tables are
        # signature-sorted first so that tiles are homogeneous and most offsets drop out
        if sig_sort_enabled(nbr) or nbr._steady.get((K, N), (None, False))[1]:
            tab, perm, masks = nbr.signature_sorted()
        else:
            tab, perm, masks = nbr.t, None, nbr.tile_masks()
        _lib.check(L.fvdb_conv_gather_tc2(x.data_ptr(), x.shape[0], K, img.data_ptr(), N, tab.data_ptr(), nbr.ld,
                                          n_out, _lib.ptr(perm), masks.data_ptr(), out.data_ptr(),
                                          _dtype_code(out_dtype), st), "conv_gather_tc")
    return out


WG_PAIRS_BELOW_DENSITY = 11.0  # mean pairs per output row under which the pair-list wgrad runs


# int32 positions inside the pair lists, kmap_compact and the halo plan's tile bases (27 * rows + padding)
INT32_ROWS_LIMIT = (2 ** 31 - 27 * 128) // 27


def wgrad_pairs_enabled(nbr: "NbrTable", cin: int, cout: int) -> bool:
    """Run the bf16 weight gradient over per-offset pair lists (fvdb_conv_wgrad_pairs_tc)?

    The table kernel (fvdb_conv_wgrad_tc) processes 27 rows per output row whatever the density. Missing
    neighbours cost it MMAs on zeros but no memory reads, and each grad_out row is shared by the CTA's
    offsets. The pair-list kernel issues MMAs for the pairs only, but gathers both operand rows per pair.
    Measured on B200 (tools/wgrad_pairs_bench.py, ms per wgrad, table vs pairs with a 6-stage ring):
    - LiDAR 128x128 (9.2 pairs/row): 0.140 vs 0.108;
    - LiDAR 64x128: 0.095 vs 0.093;
    - LiDAR 128x64: 0.103 vs 0.093;
    - cfg4 stride-2 64x128 (16.6 pairs/row): 0.120 vs 0.193;
    - shell 128x128 (20.9 pairs/row): 0.83 vs 1.39.
    Building the lists costs 0.1-0.26 ms per table (cached on it).
    Default: tables below ``WG_PAIRS_BELOW_DENSITY`` mean pairs per row, from their third wgrad on, so
    the list build and the density read-back are paid only by reused tables (a U-Net stage that rebuilds
    its maps runs two wgrads per map). It needs a 128-channel side (Cin or Cout = 128, the other 32/64/128).
    Env FVDB_WG_PAIRS: "0" never, "force" whenever the shape allows.
    """
    if not ((cin == 128 and cout in (32, 64, 128)) or (cout == 128 and cin in (32, 64, 128))):
        return False
    if nbr.n >= INT32_ROWS_LIMIT:
        return False
    v = os.environ.get("FVDB_WG_PAIRS")
    if v == "0":
        return False
    if v == "force":
        return True
    if nbr._pairs is None and nbr.wgrad_uses < 2:  # the density check reads counts back (one sync per table)
        return False
    return nbr.n > 0 and nbr.density() < WG_PAIRS_BELOW_DENSITY


def wgrad_halo_enabled(nbr: "NbrTable", cin: int, cout: int) -> bool:
    """Run the bf16 weight gradient on the table's halo plan (fvdb_conv_wgrad_halo, Cin = Cout = 32)?

    The table kernel is bound by shared memory at 32x32 (per 16-cycle MMA it writes the gathered 4 KB A block
    and reads it back with B); the halo form builds A = xᵀ in TMEM from the staged halo, so an MMA reads only B
    from shared memory.  Measured on B200 (cfg5, bench.py): 3.59 ms vs 2.83 for the table kernel -- its
    hand-off skeleton alone (FVDB_DEBUG_WGH=15: no MMA, no A build, no loads) takes 2.0 ms, so it is opt-in.
    Env FVDB_WG_HALO: "force" whenever the shape allows (the table's own plan is built if missing), else never.
    """
    if cin != 32 or cout != 32 or nbr.n >= INT32_ROWS_LIMIT:
        return False
    return os.environ.get("FVDB_WG_HALO") == "force"


def wgrad(x: torch.Tensor, go: torch.Tensor, nbr: NbrTable) -> torch.Tensor:
    """gw[co][ci][d] = Σ_o go[o,co]·x[nbr[d][o],ci]  → [Cout, Cin, 3, 3, 3] (fp32 for bf16 inputs)."""
    n_out = nbr.n
    cin, cout = int(x.shape[1]), int(go.shape[1])
    if x.dtype == torch.bfloat16 and max(cin, cout) > TC_CHANNELS[-1]:  # channel blocks (independent)
        b = TC_CHANNELS[-1]
        gw = torch.empty((cout, cin, 3, 3, 3), dtype=torch.float32, device=x.device)
        for c0 in range(0, cout, b):
            for i0 in range(0, cin, b):
                gw[c0:c0 + b, i0:i0 + b] = wgrad(x[:, i0:i0 + b], go[:, c0:c0 + b], nbr)
        return gw
    L = _lib.lib()
    st = _lib.stream_ptr()
    x, go = x.contiguous(), go.contiguous()
    if x.dtype in (torch.float32, torch.float64):
        gw = torch.empty((cout, cin, 3, 3, 3), dtype=x.dtype, device=x.device)
        code = _dtype_code(x.dtype)
        wsb = L.fvdb_wgrad_workspace_bytes(code, n_out, cin, cout)
        ws = _lib.workspace(wsb, x.device)
        _lib.check(L.fvdb_conv_wgrad_simt(code, x.data_ptr(), x.shape[0], cin, go.data_ptr(), cout, nbr.t.data_ptr(),
                                          nbr.ld, n_out, gw.data_ptr(), ws.data_ptr(), wsb, st), "conv_wgrad_simt")
        return gw
    ci_p, co_p = _tc_width(cin), _tc_width(cout)
    if (ci_p, co_p) != (cin, cout):
        gw = wgrad(_pad_cols(x, ci_p), _pad_cols(go, co_p), nbr)
        return gw[:cout, :cin].contiguous()
    gw = torch.empty((cout, cin, 3, 3, 3), dtype=torch.float32, device=x.device)
    if wgrad_halo_enabled(nbr, cin, cout):  # xᵀ in TMEM from the table's halo plan (csrc/conv_halo.cu)
        nbr.wgrad_uses += 1
        plan = nbr.halo_plan(cin, cout)
        wsb = L.fvdb_wgrad_halo_workspace_bytes(n_out)
        ws = _lib.workspace(wsb, x.device)
        _lib.check(L.fvdb_conv_wgrad_halo(x.data_ptr(), x.shape[0], cin, go.data_ptr(), cout, C.byref(plan.c), n_out,
                                          gw.data_ptr(), ws.data_ptr(), wsb, st), "conv_wgrad_halo")
        return gw
    use_pairs = wgrad_pairs_enabled(nbr, cin, cout)
    nbr.wgrad_uses += 1
    if use_pairs:
        pin, pout, seg, _ = nbr.pair_lists()
        tp = nbr.pair_tile_pos() if _WG_PAIRS_SCHED == "tiles" else None
        wsb = L.fvdb_wgrad_pairs_workspace_bytes(cin, cout, n_out)
        ws = _lib.workspace(wsb, x.device)
        _lib.check(L.fvdb_conv_wgrad_pairs_tc(x.data_ptr(), x.shape[0], cin, go.data_ptr(), cout, pin.data_ptr(),
                                              pout.data_ptr(), seg.data_ptr(), None if tp is None else tp.data_ptr(),
                                              n_out, gw.data_ptr(), ws.data_ptr(), wsb, st), "conv_wgrad_pairs_tc")
        return gw
    wsb = L.fvdb_wgrad_tc_workspace_bytes(n_out, cin, cout)
    ws = _lib.workspace(wsb, x.device)
    _lib.check(L.fvdb_conv_wgrad_tc(x.data_ptr(), x.shape[0], cin, go.data_ptr(), cout, nbr.t.data_ptr(), nbr.ld,
                                    n_out, gw.data_ptr(), ws.data_ptr(), wsb, st), "conv_wgrad_tc")
    return gw


def lggs_stats(nbr: torch.Tensor, stats: dict):  # nbr: [27, n_out] view
    """LGGS instrumentation counters (conv.py:264-301): 64-row blocks, per-offset pad to 16."""
    n = int(nbr.shape[1])
    nblocks = (n + LGGS_BLOCK - 1) // LGGS_BLOCK
    valid = (nbr >= 0).to(torch.int32)
    pad = nblocks * LGGS_BLOCK - n
    if pad:
        valid = torch.nn.functional.pad(valid, (0, pad))
    cnt = valid.reshape(27, nblocks, LGGS_BLOCK).sum(-1)
    pads = (-cnt) % LGGS_PAD
    stats["lggs_blocks"] = nblocks
    stats["lggs_pad_rows_total"] = int(pads.sum().item())
    stats["lggs_pad_rows_max"] = int(pads.max().item()) if pads.numel() else 0


# ---------------------------------------------------------------------------
# reference-compatible functional API
# ---------------------------------------------------------------------------

def variant_impl(variant, dtype):
    """Tensor-core kernel a reference ``variant`` selects (conv.py:125-261), or None for the reuse policy.

    The reference's dense-window schedules ``leaf`` (10^3 windows per leaf) and ``brick`` (6x4x4 -> 4x2x2) are
    its answer to occupied leaves; here that role is the halo-staged kernel, which stages each 128-row tile's
    exact neighbourhood in shared memory once (a window fitted to the data instead of a fixed box) and builds
    every offset's operand from it: ``leaf`` / ``brick`` run it from the first call (building the tile plan).
    ``igemm`` / ``lggs`` (gather-GEMM-scatter) keep the reuse policy (``conv_impl``): the gather kernel for a
    map's first uses, then the steady kernel (``auto-reuse``: without ``auto``'s first-use halo for shared plans).  Measured on B200 (bench.py --config dense*, fwd ms): dense 128^3
    at 64 ch, gather 1.30 vs halo 0.64."""
    if dtype == torch.bfloat16 and variant in ("leaf", "brick"):
        return "halo"
    return "auto-reuse" if conv_impl() == "auto" else None


def conv(grid_in, features, kernel, grid_out=None, variant="igemm", stride=1, kmap=None, stats=None):
    """Sparse convolution out[o] = Σ_d W[:, :, d] @ in[stride·o + d] (conv.py:136-177)."""
    stride = int(stride)
    weights = _kernel_weights(kernel)
    dev = grid_in.device
    features = _to_device_tensor(features, dev)
    w_shape = tuple(weights.shape)
    if features.ndim != 2 or features.shape[0] != grid_in.num_voxels:
        raise ValueError(f"features must be [{grid_in.num_voxels}, C_in], got {tuple(features.shape)}")
    if features.shape[1] != w_shape[1]:
        raise ValueError(f"feature channels {features.shape[1]} != kernel C_in {w_shape[1]}")
    if len(w_shape) != 5 or w_shape[2:] != (3, 3, 3):
        raise ValueError(f"kernel weights must be [C_out, C_in, 3, 3, 3], got {w_shape}")
    if grid_out is None:
        grid_out = grid_in if stride == 1 else _coarsen_grid(grid_in, 2)
    if variant == "auto":
        variant = choose_variant(grid_in, w_shape[1], w_shape[0])
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}; expected one of {VARIANTS}")
    if variant != "igemm" and stride != 1:
        raise ValueError(f"variant {variant!r} supports stride 1 only (got stride {stride})")
    _dtype_code(features.dtype)
    w = _to_device_tensor(weights, dev)
    if features.dtype != torch.bfloat16:
        w = w.to(features.dtype)  # conv.py:164
    if kmap is None:
        kmap = build_kernel_map(grid_in, grid_out, stride)
    out = gather_conv(features, kmap.fwd, w, transpose=False, impl=variant_impl(variant, features.dtype))
    if variant == "lggs" and stats is not None:
        lggs_stats(kmap.nbr, stats)
    return out


def conv_backward(kmap, grad_out, features_in, kernel):
    """(grad_in, grad_kernel) of the forward (conv.py:339-368)."""
    weights = _kernel_weights(kernel)
    dev = kmap.device
    grad_out = _to_device_tensor(grad_out, dev)
    features_in = _to_device_tensor(features_in, dev)
    c_out, c_in = int(weights.shape[0]), int(weights.shape[1])
    if tuple(grad_out.shape) != (kmap.num_out, c_out):
        raise ValueError(f"grad_out must be [{kmap.num_out}, {c_out}], got {tuple(grad_out.shape)}")
    if tuple(features_in.shape) != (kmap.num_in, c_in):
        raise ValueError(f"features_in must be [{kmap.num_in}, {c_in}], got {tuple(features_in.shape)}")
    w = _to_device_tensor(weights, dev)
    w_dtype = w.dtype
    if grad_out.dtype != torch.bfloat16:
        w = w.to(grad_out.dtype)
    grad_in = gather_conv(grad_out, kmap.bwd, w, transpose=True,
                          out_dtype=features_in.dtype if features_in.dtype == torch.bfloat16 else None)
    grad_in = grad_in.to(features_in.dtype)
    gw = wgrad(features_in.to(grad_out.dtype) if grad_out.dtype != torch.bfloat16 else features_in.to(torch.bfloat16),
               grad_out, kmap.fwd)
    return grad_in, gw.to(w_dtype)


def conv_transpose(kmap, x_coarse, kernel, out_dtype=None):
    """Transposed (stride-2 adjoint) conv, SURVEY §8.0 C7.

    y[i] = Σ_d Σ_{(i,o)∈K_d} x_coarse[o] @ W_d  with ``kernel`` [C_coarse, C_fine, 3, 3, 3]
    (PyTorch ConvTranspose orientation) and ``kmap`` the stride-2 fine→coarse map.
    Equals ``conv_backward(kmap, x_coarse, 0, kernel)[0]``.
    """
    weights = _kernel_weights(kernel)
    dev = kmap.device
    x = _to_device_tensor(x_coarse, dev)
    if tuple(x.shape) != (kmap.num_out, int(weights.shape[0])):
        raise ValueError(f"x_coarse must be [{kmap.num_out}, {int(weights.shape[0])}], got {tuple(x.shape)}")
    w = _to_device_tensor(weights, dev)
    if x.dtype != torch.bfloat16:
        w = w.to(x.dtype)
    return gather_conv(x, kmap.bwd, w, transpose=True, out_dtype=out_dtype)


def conv_batch(batch, features, kernel, variant="igemm"):
    """Stride-1 convolution per batch element, one launch for the batch (conv.py:371-383)."""
    from .jagged import GridBatch
    if not isinstance(batch, GridBatch):
        raise TypeError("conv_batch needs a GridBatch; use conv() for a single grid")
    feats = _to_device_tensor(batch.check_features(features), batch.device)
    weights = _kernel_weights(kernel)
    if variant == "auto":
        variant = choose_variant(batch.grids[0], int(weights.shape[1]), int(weights.shape[0]))
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}; expected one of {VARIANTS}")
    if feats.shape[1] != int(weights.shape[1]):
        raise ValueError(f"feature channels {feats.shape[1]} != kernel C_in {int(weights.shape[1])}")
    km = batch_grid_kernel_map(batch, batch, 1)
    w = _to_device_tensor(weights, feats.device)
    if feats.dtype != torch.bfloat16:
        w = w.to(feats.dtype)
    return batch.jagged(gather_conv(feats, km.fwd, w, impl=variant_impl(variant, feats.dtype)))


def cache_batch_kernel_map(batch_in, batch_out, stride, km):
    """Store ``km`` as the (batch_in -> batch_out, stride) map in ``batch_out``'s cache.

    The entry is keyed by the ids of ``batch_in``'s grids and holds weak references to them that every lookup
    checks, so grids that reuse a collected grid's id never get the old map; entries of collected grids are
    dropped on the next store.  No strong reference from the cache back to the grids: no cycles."""
    cache = batch_out._kmaps
    for k in [k for k, v in cache.items() if k[0] == "kmap" and any(r() is None for r in v[0])]:  # noqa: E501
        del cache[k]
    cache[("kmap", tuple(id(g) for g in batch_in.grids), int(stride))] = (
        tuple(weakref.ref(g) for g in batch_in.grids), km)
    return km


def cached_batch_kernel_map(batch_in, batch_out, stride):
    v = batch_out._kmaps.get(("kmap", tuple(id(g) for g in batch_in.grids), int(stride)))
    if v is not None and all(r() is g for r, g in zip(v[0], batch_in.grids)):
        return v[1]
    return None


def batch_grid_kernel_map(batch_in, batch_out, stride):
    """Batch-global kernel map of two aligned GridBatches (cached on ``batch_out``)."""
    km = cached_batch_kernel_map(batch_in, batch_out, stride)
    if km is not None:
        return km
    if len(batch_in.grids) != len(batch_out.grids):
        raise ValueError(f"grid batches differ in size: {len(batch_in.grids)} vs {len(batch_out.grids)}")
    if len(batch_in.grids) == 1:
        km = build_kernel_map(batch_in.grids[0], batch_out.grids[0], stride)
    else:
        km = build_batch_kernel_map(batch_in, batch_out, stride)
    return cache_batch_kernel_map(batch_in, batch_out, stride, km)


# ---------------------------------------------------------------------------
# U-Net glue: pool / upsample_nearest (conv.py:386-446)
# ---------------------------------------------------------------------------

def _floor_div(coords: torch.Tensor, factor: int) -> torch.Tensor:
    if factor == 1 or coords.shape[0] == 0:
        return coords
    out = torch.empty_like(coords)
    _lib.check(_lib.lib().fvdb_floor_div_coords(coords.data_ptr(), coords.shape[0], int(factor), out.data_ptr(),
                                                _lib.stream_ptr()), "floor_div")
    return out


def pool(grid, features, factor, mode="avg"):
    """Reduce features onto the coarsened grid over active fine children only (conv.py:401-426).

    ``avg`` divides by the count of active children (not factor^3), accumulating in float64 in the
    reference's order; ``max`` takes their componentwise maximum.  Returns (coarse_grid, coarse_features).
    """
    if mode not in ("avg", "max"):
        raise ValueError(f"pool mode must be 'avg' or 'max', got {mode!r}")
    factor = int(factor)
    dev = grid.device
    feats = _to_device_tensor(features, dev)
    if feats.shape[0] != grid.num_voxels:
        raise ValueError(f"features rows {feats.shape[0]} != voxel count {grid.num_voxels}")
    coarse = _coarsen_grid(grid, factor)
    if factor == 1:
        return coarse, feats.clone()
    prow = coarse.coord_to_index_many(_floor_div(grid.active_coords(), factor))
    chans = int(np.prod(feats.shape[1:])) if feats.ndim > 1 else 1
    out = torch.empty((coarse.num_voxels,) + tuple(feats.shape[1:]), dtype=feats.dtype, device=dev)
    if grid.num_voxels:
        L = _lib.lib()
        wsb = L.fvdb_pool_workspace_bytes(grid.num_voxels, coarse.num_voxels)
        ws = _lib.workspace(wsb, dev)
        detail = C.c_int64(-1)
        f = feats.contiguous()
        _lib.check(L.fvdb_pool(_dtype_code(f.dtype), f.data_ptr(), grid.num_voxels, chans, prow.data_ptr(),
                               coarse.num_voxels, int(mode == "max"), out.data_ptr(), C.byref(detail),
                               ws.data_ptr(), wsb, _lib.stream_ptr()), "pool")
    return coarse, out


def upsample_nearest(coarse_grid, features, factor, fine_grid):
    """Copy each fine active voxel's feature from its floor-division parent (conv.py:429-446)."""
    factor = int(factor)
    dev = fine_grid.device
    feats = _to_device_tensor(features, dev).contiguous()
    if feats.shape[0] != coarse_grid.num_voxels:
        raise ValueError(
            f"features rows {feats.shape[0]} != coarse voxel count {coarse_grid.num_voxels}")
    fine_coords = fine_grid.active_coords()
    prow = coarse_grid.coord_to_index_many(_floor_div(fine_coords, factor) if factor > 1 else fine_coords)
    out = torch.empty((fine_grid.num_voxels,) + tuple(feats.shape[1:]), dtype=feats.dtype, device=dev)
    n = fine_grid.num_voxels
    if n:
        L = _lib.lib()
        ws = _lib.workspace(256, dev)
        detail = C.c_int64(-1)
        row_bytes = feats[0].numel() * feats.element_size() if feats.shape[0] else 1
        rc = L.fvdb_gather_rows(feats.data_ptr(), row_bytes, prow.data_ptr(), n, out.data_ptr(), C.byref(detail),
                                ws.data_ptr(), 256, _lib.stream_ptr())
        if rc == _lib.FVDB_ERR_INVALID and detail.value >= 0:
            bad = fine_coords[int(detail.value)].tolist()
            raise ValueError(f"fine voxel {tuple(bad)} has no active parent")
        _lib.check(rc, "upsample_nearest")
    return out


def pool_batch(batch, features, factor, mode="avg"):
    """Pooling applied per batch element; returns (coarse GridBatch, features) (conv.py:386-398)."""
    from .jagged import GridBatch
    if not isinstance(batch, GridBatch):
        raise TypeError("pool_batch needs a GridBatch; use pool() for a single grid")
    feats = _to_device_tensor(batch.check_features(features), batch.device)
    coarse, parts = [], []
    for b, g in enumerate(batch.grids):
        cg, cf = pool(g, feats[batch.voxel_slice(b)], factor, mode)
        coarse.append(cg)
        parts.append(cf)
    out = GridBatch(coarse)
    return out, out.jagged(torch.cat(parts, 0))
