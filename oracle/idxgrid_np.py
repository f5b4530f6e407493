"""numpy restatement of the reference index-grid / sparse-conv algorithms.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Citations are to the
reference checkout, ``pkg/src/idxgrid/<file>:<line>``.

The restatement is deliberately written from the *specification* of each step
(key layouts, ordering, rank arithmetic) rather than transcribed: e.g. the
reference's four-pass 16-bit LSD radix argsort (build.py:51-61) is restated as
one stable argsort on the full 64-bit key, which yields the identical
permutation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "COORD_LIMIT", "ROOT_TABLE_LIMIT", "STENCIL", "OGrid",
    "tile_key_u64", "upper_off", "lower_off", "leaf_off", "voxel_key_u64",
    "quantize", "build_from_coords", "build_from_points", "coarsen", "empty",
    "coord_to_index", "active_coords", "kernel_map", "kernel_map_table",
    "conv_igemm", "conv_backward", "conv_transpose", "conv_dense",
    "subdivide", "dilate", "pool", "upsample_nearest", "interp_stencil", "sample", "splat",
]

COORD_LIMIT = 1 << 30          # topology.py:24
ROOT_TABLE_LIMIT = 1 << 28     # build.py:32

# stencil offsets, di slowest (conv.py:36-38); offset index (di+1)*9+(dj+1)*3+(dk+1) (conv.py:100-102)
STENCIL = np.array([(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)],
                   dtype=np.int64)

_M21 = np.int64(0x1FFFFF)


# ---------------------------------------------------------------------------
# key layouts (topology.py:47-59, 83-93; build.py:74-79)
# ---------------------------------------------------------------------------

def tile_key_u64(c):
    """63-bit root key of each coordinate's 4096³ tile (topology.py:83-88)."""
    c = np.asarray(c, np.int64)
    f = (c >> 12) & _M21
    return ((f[:, 0].astype(np.uint64) << np.uint64(42))
            | (f[:, 1].astype(np.uint64) << np.uint64(21))
            | f[:, 2].astype(np.uint64))


def upper_off(c):
    """Child slot of the 128³ lower node inside its 32³ upper node (topology.py:57-59)."""
    c = np.asarray(c, np.int64)
    u = (c & 4095) >> 7
    return (u[:, 0] << 10) | (u[:, 1] << 5) | u[:, 2]


def lower_off(c):
    """Child slot of the 8³ leaf inside its 16³ lower node (topology.py:52-54)."""
    c = np.asarray(c, np.int64)
    u = (c & 127) >> 3
    return (u[:, 0] << 8) | (u[:, 1] << 4) | u[:, 2]


def leaf_off(c):
    """Bit position of a voxel inside its 8³ leaf (topology.py:47-49)."""
    c = np.asarray(c, np.int64)
    u = c & 7
    return (u[:, 0] << 6) | (u[:, 1] << 3) | u[:, 2]


def voxel_key_u64(tile_rank, c):
    """run<<36 | upper<<21 | lower<<9 | leaf (build.py:74-79)."""
    low = (upper_off(c) << 21) | (lower_off(c) << 9) | leaf_off(c)
    return (np.asarray(tile_rank, np.uint64) << np.uint64(36)) | low.astype(np.uint64)


# ---------------------------------------------------------------------------
# grid container (topology.py:140-201)
# ---------------------------------------------------------------------------

@dataclass
class OGrid:
    tile_keys: np.ndarray            # [Ut] uint64
    upper_origins: np.ndarray        # [Ut,3] int64
    upper_child_starts: np.ndarray   # [Ut+1] int64
    lower_offset_in_upper: np.ndarray  # [Lo] uint16
    lower_origins: np.ndarray        # [Lo,3] int64
    lower_child_starts: np.ndarray   # [Lo+1] int64
    leaf_offset_in_lower: np.ndarray  # [L] uint16
    leaf_keys: np.ndarray            # [L] uint64
    leaf_origins: np.ndarray         # [L,3] int64
    leaf_masks: np.ndarray           # [L,8] uint64
    leaf_prefix: np.ndarray          # [L] uint64
    leaf_value_offset: np.ndarray    # [L] uint64
    num_voxels: int
    voxel_size: np.ndarray
    origin: np.ndarray

    @property
    def counts(self):
        return (len(self.tile_keys), len(self.lower_origins), len(self.leaf_origins),
                self.num_voxels)

    @property
    def num_leaf_nodes(self):
        return len(self.leaf_origins)

    def leaf_occupancy(self):
        return 0.0 if self.num_leaf_nodes == 0 else self.num_voxels / (512.0 * self.num_leaf_nodes)


ARRAY_FIELDS = ("tile_keys", "upper_origins", "upper_child_starts", "lower_offset_in_upper",
                "lower_origins", "lower_child_starts", "leaf_offset_in_lower", "leaf_keys",
                "leaf_origins", "leaf_masks", "leaf_prefix", "leaf_value_offset")


def empty(voxel_size=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0)):
    """Grid with no active voxels (topology.py:386-404)."""
    z3 = np.zeros((0, 3), np.int64)
    return OGrid(np.zeros(0, np.uint64), z3, np.zeros(1, np.int64), np.zeros(0, np.uint16),
                 z3.copy(), np.zeros(1, np.int64), np.zeros(0, np.uint16), np.zeros(0, np.uint64),
                 z3.copy(), np.zeros((0, 8), np.uint64), np.zeros(0, np.uint64),
                 np.zeros(0, np.uint64), 0, np.asarray(voxel_size, np.float64).reshape(3),
                 np.asarray(origin, np.float64).reshape(3))


# ---------------------------------------------------------------------------
# construction (build.py:82-230, 325-339; topology.py:135-137)
# ---------------------------------------------------------------------------

def quantize(points, voxel_size, origin):
    """floor((p - origin)/vs + 0.5) in float64 (topology.py:128-137)."""
    p = np.asarray(points, np.float64).reshape(-1, 3)
    q = (p - np.asarray(origin, np.float64)) / np.asarray(voxel_size, np.float64)
    return np.floor(q + 0.5).astype(np.int64)


def _segments(sorted_vals):
    """(values, first-index, run length) of the equal runs of a sorted array (build.py:64-71)."""
    n = len(sorted_vals)
    if n == 0:
        return sorted_vals[:0], np.zeros(0, np.int64), np.zeros(0, np.int64)
    head = np.ones(n, bool)
    head[1:] = sorted_vals[1:] != sorted_vals[:-1]
    first = np.flatnonzero(head)
    return sorted_vals[first], first, np.diff(np.append(first, n))


def build_from_coords(coords, voxel_size=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0)):
    """Sort/RLE grid build (build.py:82-142) + node registration (build.py:145-198).

    Raises ValueError with the reference's messages (build.py:96-101, 121-122).
    """
    c = np.asarray(coords, np.int64).reshape(-1, 3)
    if len(c) == 0:
        return empty(voxel_size, origin)
    bad_rows = np.flatnonzero((np.abs(c) > COORD_LIMIT).any(axis=1))
    if len(bad_rows):
        r = int(bad_rows[0])
        raise ValueError(f"coordinate out of range at row {r}: {tuple(c[r].tolist())} "
                         f"(components must be within +-{COORD_LIMIT})")
    # tile ranks: unique sorted tile keys (the stable radix sort + RLE of build.py:111-124)
    tk = tile_key_u64(c)
    tiles, inv = np.unique(tk, return_inverse=True)
    if len(tiles) > ROOT_TABLE_LIMIT:
        raise ValueError(f"root table limit exceeded: {len(tiles)} tiles > {ROOT_TABLE_LIMIT}")
    # one sort of the per-run voxel keys, then dedupe (build.py:126-134)
    vk = voxel_key_u64(inv.astype(np.int64), c)
    vk = np.sort(vk, kind="stable")
    uvox, _, _ = _segments(vk)
    return _register(tiles, uvox, voxel_size, origin)


def _register(tiles, uvox, voxel_size, origin):
    """Node registration from sorted unique voxel keys (build.py:145-198)."""
    leaf_vals, _, leaf_pop = _segments(uvox >> np.uint64(9))
    lower_vals, _, lower_nleaf = _segments(leaf_vals >> np.uint64(12))
    upper_vals, _, upper_nlower = _segments(lower_vals >> np.uint64(15))
    n_leaf, n_lower = len(leaf_vals), len(lower_vals)
    assert len(upper_vals) == len(tiles)

    # occupancy bits, one per voxel; leaves are contiguous runs of uvox (build.py:153-159)
    leaf_id = np.repeat(np.arange(n_leaf), leaf_pop)
    pos = (uvox & np.uint64(511)).astype(np.int64)
    bits = np.zeros((n_leaf, 512), bool)
    bits[leaf_id, pos] = True
    packed = np.packbits(bits, axis=1, bitorder="little")          # [L, 64] bytes, bit m at byte m>>3
    masks = np.ascontiguousarray(packed).view("<u8").reshape(n_leaf, 8).astype(np.uint64)

    # 9-bit cumulative popcount fields of words 0..6 (build.py:161-166)
    pops = np.bitwise_count(masks).astype(np.int64)
    cum = np.cumsum(pops, axis=1)
    prefix = np.zeros(n_leaf, np.uint64)
    for t in range(7):
        prefix |= cum[:, t].astype(np.uint64) << np.uint64(9 * t)
    # value offsets = 1 + exclusive scan of leaf popcounts (build.py:167-170)
    vo = np.ones(n_leaf, np.int64)
    vo[1:] += np.cumsum(cum[:, 7])[:-1]

    # origins top-down (build.py:172-182; topology.py:96-103; build.py:201-216)
    fields = np.stack([(tiles >> np.uint64(s)) & np.uint64(0x1FFFFF) for s in (42, 21, 0)], 1)
    f = fields.astype(np.int64)
    up_orig = np.where(f >= (1 << 20), f - (1 << 21), f) << 12
    lo_local = (lower_vals & np.uint64(0x7FFF)).astype(np.int64)
    lo_orig = np.repeat(up_orig, upper_nlower, axis=0) + (np.stack(
        [(lo_local >> 10) & 31, (lo_local >> 5) & 31, lo_local & 31], 1) << 7)
    lf_local = (leaf_vals & np.uint64(0xFFF)).astype(np.int64)
    lf_orig = np.repeat(lo_orig, lower_nleaf, axis=0) + (np.stack(
        [(lf_local >> 8) & 15, (lf_local >> 4) & 15, lf_local & 15], 1) << 3)

    def starts(cnt):
        return np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)

    return OGrid(tiles.astype(np.uint64), up_orig, starts(upper_nlower),
                 lo_local.astype(np.uint16), lo_orig, starts(lower_nleaf),
                 lf_local.astype(np.uint16), leaf_vals.astype(np.uint64), lf_orig, masks,
                 prefix, vo.astype(np.uint64), int(len(uvox)),
                 np.asarray(voxel_size, np.float64).reshape(3),
                 np.asarray(origin, np.float64).reshape(3))


def build_from_points(points, voxel_size, origin):
    """Finite check then quantize then build (build.py:219-230)."""
    p = np.asarray(points, np.float64).reshape(-1, 3)
    bad = np.flatnonzero(~np.isfinite(p).all(axis=1))
    if len(bad):
        r = int(bad[0])
        raise ValueError(f"non-finite point at row {r}: {p[r].tolist()}")
    return build_from_coords(quantize(p, voxel_size, origin), voxel_size, origin)


def coarsen(grid, factor):
    """Coarse voxel active iff any fine child is (build.py:325-339)."""
    factor = int(factor)
    if factor < 1:
        raise ValueError("coarsening factor must be >= 1")
    c = active_coords(grid)
    vs, og = grid.voxel_size, grid.origin
    if factor > 1:
        c = np.floor_divide(c, factor)
        og = og + vs * (factor - 1) / 2.0
        vs = vs * factor
    if len(c) == 0:
        return empty(vs, og)
    return build_from_coords(c, vs, og)


# ---------------------------------------------------------------------------
# queries (topology.py:253-299)
# ---------------------------------------------------------------------------

def coord_to_index(grid, coords):
    """1-based index of each coord, 0 for background (topology.py:253-286)."""
    c = np.asarray(coords, np.int64).reshape(-1, 3)
    out = np.zeros(len(c), np.int64)
    if len(c) == 0 or grid.num_leaf_nodes == 0:
        return out
    tk = tile_key_u64(c)
    t = np.searchsorted(grid.tile_keys, tk)
    t = np.minimum(t, len(grid.tile_keys) - 1)
    hit = grid.tile_keys[t] == tk
    lk = (t.astype(np.uint64) << np.uint64(27)) | ((upper_off(c) << 12) | lower_off(c)).astype(np.uint64)
    leaf = np.minimum(np.searchsorted(grid.leaf_keys, lk), grid.num_leaf_nodes - 1)
    hit &= grid.leaf_keys[leaf] == lk
    m = leaf_off(c)
    w = m >> 6
    word = grid.leaf_masks[leaf, w]
    b = (m & 63).astype(np.uint64)
    hit &= ((word >> b) & np.uint64(1)) == 1
    below = (grid.leaf_prefix[leaf] >> (np.maximum(w - 1, 0).astype(np.uint64) * np.uint64(9))) & np.uint64(511)
    below = np.where(w > 0, below.astype(np.int64), 0)
    rank = np.bitwise_count(word & ((np.uint64(1) << b) - np.uint64(1))).astype(np.int64)
    idx = grid.leaf_value_offset[leaf].astype(np.int64) + below + rank
    out[hit] = idx[hit]
    return out


def active_coords(grid):
    """[N,3] coordinates in index order (topology.py:288-299)."""
    if grid.num_leaf_nodes == 0:
        return np.zeros((0, 3), np.int64)
    bits = np.unpackbits(grid.leaf_masks.astype("<u8").view(np.uint8), bitorder="little")
    leaf, m = np.nonzero(bits.reshape(grid.num_leaf_nodes, 512))
    local = np.stack([m >> 6, (m >> 3) & 7, m & 7], 1).astype(np.int64)
    return grid.leaf_origins[leaf] + local


# ---------------------------------------------------------------------------
# kernel map + convolution (conv.py:80-122, 136-191, 304-368)
# ---------------------------------------------------------------------------

def kernel_map(grid_in, grid_out, stride=1):
    """Per-offset (in_rows, out_rows) int64, out ascending (conv.py:105-122)."""
    stride = int(stride)
    if stride not in (1, 2):
        raise ValueError(f"stride must be 1 or 2, got {stride}")
    oc = active_coords(grid_out)
    rows = np.arange(len(oc), dtype=np.int64)
    ins, outs = [], []
    for d in STENCIL:
        idx = coord_to_index(grid_in, stride * oc + d)
        keep = idx > 0
        ins.append(idx[keep] - 1)
        outs.append(rows[keep])
    return ins, outs


def kernel_map_table(ins, outs, n_out):
    """Dense [27, n_out] int32 neighbour table (-1 = none) from the per-offset lists."""
    t = np.full((27, n_out), -1, np.int64)
    for d in range(27):
        t[d, outs[d]] = ins[d]
    return t


def conv_igemm(features, weights, ins, outs, n_out):
    """Gather-GEMM-scatter forward, out[o] = Σ_d W_d @ in[s·o+d] (conv.py:180-191)."""
    f = np.asarray(features)
    w = np.asarray(weights).astype(f.dtype, copy=False)
    out = np.zeros((n_out, w.shape[0]), f.dtype)
    for d, (a, b, c) in enumerate(STENCIL):
        if len(outs[d]):
            out[outs[d]] += f[ins[d]] @ w[:, :, a + 1, b + 1, c + 1].T
    return out


def conv_backward(ins, outs, grad_out, features, weights):
    """(grad_in, grad_w) of the igemm forward (conv.py:339-368)."""
    go = np.asarray(grad_out)
    f = np.asarray(features)
    w = np.asarray(weights)
    gi = np.zeros_like(f)
    gw = np.zeros_like(w)
    for d, (a, b, c) in enumerate(STENCIL):
        if len(outs[d]) == 0:
            continue
        g = go[outs[d]]
        gi[ins[d]] += g @ w[:, :, a + 1, b + 1, c + 1].astype(go.dtype, copy=False)
        gw[:, :, a + 1, b + 1, c + 1] = g.T @ f[ins[d]]
    return gi, gw


def conv_transpose(ins, outs, x_coarse, weights, n_fine):
    """Transposed (stride-2 adjoint) conv: y[i] = Σ_d Σ_{(i,o)∈K_d} x[o] @ W_d.

    Derived from conv.py:339-368: conv_backward(K, x, 0, W)[0].
    ``weights`` is [C_coarse, C_fine, 3, 3, 3].
    """
    x = np.asarray(x_coarse)
    w = np.asarray(weights).astype(x.dtype, copy=False)
    y = np.zeros((n_fine, w.shape[1]), x.dtype)
    for d, (a, b, c) in enumerate(STENCIL):
        if len(outs[d]):
            y[ins[d]] += x[outs[d]] @ w[:, :, a + 1, b + 1, c + 1]
    return y


def conv_dense(grid_in, features, weights, grid_out, stride=1):
    """Independent dense-box evaluation of the operator (conv.py:304-336)."""
    f = np.asarray(features)
    w = np.asarray(weights)
    ic = active_coords(grid_in)
    oc = active_coords(grid_out)
    out = np.zeros((len(oc), w.shape[0]), np.float64)
    if len(ic) == 0 or len(oc) == 0:
        return out.astype(f.dtype)
    lo = ic.min(0) - 1
    shape = tuple((ic.max(0) + 2 - lo).tolist())
    dense = np.zeros(shape + (f.shape[1],), np.float64)
    p = ic - lo
    dense[p[:, 0], p[:, 1], p[:, 2]] = f
    for d, (a, b, c) in enumerate(STENCIL):
        q = stride * oc + (a, b, c) - lo
        ok = (q >= 0).all(1) & (q < np.array(shape)).all(1)
        if ok.any():
            out[ok] += dense[q[ok, 0], q[ok, 1], q[ok, 2]] @ w[:, :, a + 1, b + 1, c + 1].astype(np.float64).T
    return out


# ---------------------------------------------------------------------------
# U-Net glue: subdivide / dilate (build.py:310-360), pool / upsample (conv.py:401-446)
# ---------------------------------------------------------------------------

def _cube(lo, width):
    r = np.arange(lo, lo + width, dtype=np.int64)
    return np.stack(np.meshgrid(r, r, r, indexing="ij"), -1).reshape(-1, 3)


def subdivide(grid, factor):
    """Every active voxel -> its factor^3 children; voxel size / factor, origin shifted (build.py:342-360)."""
    factor = int(factor)
    if factor < 1:
        raise ValueError("subdivision factor must be >= 1")
    c = active_coords(grid)
    vs, og = grid.voxel_size, grid.origin
    if factor > 1:
        vs = vs / factor
        og = og - vs * (factor - 1) / 2.0
        c = (c[:, None, :] * factor + _cube(0, factor)[None]).reshape(-1, 3)
    if len(c) == 0:
        return empty(vs, og)
    return build_from_coords(c, vs, og)


def dilate(grid, radius):
    """Union of the active set shifted by [-r, r]^3 (build.py:310-322)."""
    radius = int(radius)
    if radius < 1:
        raise ValueError("dilation radius must be >= 1")
    c = active_coords(grid)
    if len(c) == 0:
        return empty(grid.voxel_size, grid.origin)
    c = (c[:, None, :] + _cube(-radius, 2 * radius + 1)[None]).reshape(-1, 3)
    return build_from_coords(c, grid.voxel_size, grid.origin)


def pool(grid, features, factor, mode="avg"):
    """Average (float64, np.add.at row order, / active-child count) or max over active children (conv.py:401-426)."""
    if mode not in ("avg", "max"):
        raise ValueError(f"pool mode must be 'avg' or 'max', got {mode!r}")
    factor = int(factor)
    f = np.asarray(features)
    coarse = coarsen(grid, factor)
    if factor == 1:
        return coarse, f.copy()
    prow = coord_to_index(coarse, np.floor_divide(active_coords(grid), factor)) - 1
    if mode == "avg":
        acc = np.zeros((coarse.num_voxels,) + f.shape[1:], np.float64)
        np.add.at(acc, prow, f)
        cnt = np.bincount(prow, minlength=coarse.num_voxels).astype(np.float64)
        return coarse, (acc / cnt.reshape(-1, *([1] * (f.ndim - 1)))).astype(f.dtype)
    acc = np.full((coarse.num_voxels,) + f.shape[1:], -np.inf)
    np.maximum.at(acc, prow, f)
    return coarse, acc.astype(f.dtype)


def upsample_nearest(coarse, features, factor, fine):
    """Each fine voxel copies its floor-division parent's row; orphans raise (conv.py:429-446)."""
    factor = int(factor)
    fc = active_coords(fine)
    prow = coord_to_index(coarse, np.floor_divide(fc, factor) if factor > 1 else fc) - 1
    if (prow < 0).any():
        bad = fc[int(np.flatnonzero(prow < 0)[0])]
        raise ValueError(f"fine voxel {tuple(bad.tolist())} has no active parent")
    return np.asarray(features)[prow]


# ---------------------------------------------------------------------------
# grid <-> point transfer (interp.py:44-203)
# ---------------------------------------------------------------------------

def _axis_weights(u, mode):
    """Per-axis taps: trilinear 2 (floor base), bezier 3 (quadratic B-spline, round base) (interp.py:44-72)."""
    if mode == "trilinear":
        base = np.floor(u)
        f = u - base
        w = np.stack([1.0 - f, f], axis=2)
        dw = np.stack([-np.ones_like(f), np.ones_like(f)], axis=2)
        offs = np.array([0, 1], np.int64)
    else:
        base = np.floor(u + 0.5)
        offs = np.array([-1, 0, 1], np.int64)
        x = u[:, :, None] - (base[:, :, None] + offs)
        ax = np.abs(x)
        outer = np.maximum(1.5 - ax, 0.0)
        w = np.where(ax <= 0.5, 0.75 - x * x, 0.5 * outer * outer)
        dw = np.where(ax <= 0.5, -2.0 * x, -np.sign(x) * outer)
    return base.astype(np.int64), offs, w, dw


def interp_stencil(grid, points, mode):
    """rows [n,S] (-1 background), weights [n,S], world-space weight gradients [n,S,3] (interp.py:75-107)."""
    u = (np.asarray(points, np.float64) - grid.origin) / grid.voxel_size
    base, offs, w, dw = _axis_weights(u, mode)
    k = len(offs)
    sten = np.stack(np.meshgrid(offs, offs, offs, indexing="ij"), -1).reshape(-1, 3)
    rows = coord_to_index(grid, (base[:, None, :] + sten[None]).reshape(-1, 3)).reshape(len(u), -1) - 1
    wx, wy, wz = w[:, 0, :, None, None], w[:, 1, None, :, None], w[:, 2, None, None, :]
    dx, dy, dz = dw[:, 0, :, None, None], dw[:, 1, None, :, None], dw[:, 2, None, None, :]
    inv = 1.0 / grid.voxel_size
    weights = (wx * wy * wz).reshape(len(u), k ** 3)
    dweights = np.stack([(dx * wy * wz).reshape(len(u), k ** 3) * inv[0],
                         (wx * dy * wz).reshape(len(u), k ** 3) * inv[1],
                         (wx * wy * dz).reshape(len(u), k ** 3) * inv[2]], axis=2)
    return rows, weights, dweights


def sample(grid, features, points, mode="trilinear"):
    """Values [n,C] and gradients [n,C,3]: f64 sums over the stencil (interp.py:142-164)."""
    f = np.asarray(features)
    rows, w, dw = interp_stencil(grid, points, mode)
    padded = np.concatenate([f.astype(np.float64), np.zeros((1, f.shape[1]))])
    neigh = padded[rows]
    return (np.einsum("ns,nsc->nc", w, neigh).astype(f.dtype),
            np.einsum("nsx,nsc->ncx", dw, neigh).astype(f.dtype))


def splat(grid, points, point_features, mode="trilinear"):
    """Per-voxel sums of w * f over (point, tap) in stable destination order (interp.py:167-203)."""
    pf = np.asarray(point_features)
    rows, w, _ = interp_stencil(grid, points, mode)
    contrib = (w[:, :, None] * pf.astype(np.float64)[:, None, :]).reshape(-1, pf.shape[1])
    rows = rows.ravel()
    keep = rows >= 0
    rows, contrib = rows[keep], contrib[keep]
    out = np.zeros((grid.num_voxels, pf.shape[1]), np.float64)
    if len(rows):
        order = np.argsort(rows, kind="stable")
        rows, contrib = rows[order], contrib[order]
        starts = np.concatenate(([0], np.flatnonzero(rows[1:] != rows[:-1]) + 1))
        out[rows[starts]] += np.add.reduceat(contrib, starts, axis=0)
    return out.astype(pf.dtype)
