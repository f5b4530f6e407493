"""Device-resident index grid (drop-in for reference ``idxgrid.topology``).

The topology arrays are the reference's (topology.py:140-177) with identical
values, held as CUDA tensors: 64-bit unsigned arrays (``tile_keys``,
``leaf_keys``, ``leaf_masks``, ``leaf_prefix``, ``leaf_value_offset``) are stored
bit-for-bit in ``torch.int64`` and 16-bit offsets in ``torch.int16``; use
:meth:`IndexGrid.to_numpy` for the reference dtypes.  Grids are immutable.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

LEAF_SPAN = 8
LOWER_SPAN = 128
UPPER_SPAN = 4096
COORD_LIMIT = 1 << 30

ARRAY_FIELDS = ("tile_keys", "upper_origins", "upper_child_starts", "lower_offset_in_upper",
                "lower_origins", "lower_child_starts", "leaf_offset_in_lower", "leaf_keys",
                "leaf_origins", "leaf_masks", "leaf_prefix", "leaf_value_offset")
# reference dtypes (topology.py:386-404)
_NP_DTYPES = {"tile_keys": np.uint64, "upper_origins": np.int64, "upper_child_starts": np.int64,
              "lower_offset_in_upper": np.uint16, "lower_origins": np.int64,
              "lower_child_starts": np.int64, "leaf_offset_in_lower": np.uint16,
              "leaf_keys": np.uint64, "leaf_origins": np.int64, "leaf_masks": np.uint64,
              "leaf_prefix": np.uint64, "leaf_value_offset": np.uint64}
_TORCH_DTYPES = {k: (torch.int16 if v == np.uint16 else torch.int64) for k, v in _NP_DTYPES.items()}


def leaf_offset(i, j, k):
    """Linear offset inside the 8^3 leaf (topology.py:47-49)."""
    return ((i & 7) << 6) | ((j & 7) << 3) | (k & 7)


def lower_offset(i, j, k):
    """Leaf slot inside its 16^3 lower node (topology.py:52-54)."""
    return (((i & 127) >> 3) << 8) | (((j & 127) >> 3) << 4) | ((k & 127) >> 3)


def upper_offset(i, j, k):
    """Lower-node slot inside its 32^3 upper node (topology.py:57-59)."""
    return (((i & 4095) >> 7) << 10) | (((j & 4095) >> 7) << 5) | ((k & 4095) >> 7)


@dataclass(frozen=True)
class VoxelTransform:
    """World <-> index mapping; voxel (0,0,0) centred at ``origin`` (topology.py:106-137)."""

    voxel_size: np.ndarray
    origin: np.ndarray

    def __post_init__(self):
        vs = np.asarray(self.voxel_size, np.float64).reshape(3).copy()
        og = np.asarray(self.origin, np.float64).reshape(3).copy()
        if not np.all(vs > 0):
            raise ValueError(f"voxel_size must be positive, got {vs.tolist()}")
        vs.flags.writeable = False
        og.flags.writeable = False
        object.__setattr__(self, "voxel_size", vs)
        object.__setattr__(self, "origin", og)

    @staticmethod
    def uniform(size, origin=(0.0, 0.0, 0.0)):
        return VoxelTransform(np.full(3, float(size)), origin)

    def world_to_index(self, points):
        return (np.asarray(points, np.float64) - self.origin) / self.voxel_size

    def index_to_world(self, ijk):
        return np.asarray(ijk, np.float64) * self.voxel_size + self.origin

    def quantize(self, points):
        """Nearest-voxel-centre quantization on the device (same IEEE f64 ops as the reference)."""
        from .build import quantize_points
        return quantize_points(points, self)


def _device():
    _lib.lib()  # raises FvdbError without a CUDA device: there is no CPU fallback
    return torch.device("cuda", torch.cuda.current_device())


class IndexGrid:
    """Immutable sparse topology on one CUDA device (topology.py:140-305)."""

    __slots__ = ARRAY_FIELDS + ("num_voxels", "transform", "name", "_view", "_batch", "_tables", "__weakref__")

    def __init__(self, *, num_voxels, transform, name="", **arrays):
        for f in ARRAY_FIELDS:
            object.__setattr__(self, f, arrays[f])
        self.num_voxels = int(num_voxels)
        self.transform = transform
        self.name = name
        self._view = None
        self._tables = None
        self._batch = None  # kernel-map cache of the single-grid GridBatch views of this grid (as_grid_batch)

    # -- counts (topology.py:179-201) ---------------------------------------
    @property
    def device(self):
        return self.leaf_masks.device

    @property
    def num_upper_nodes(self):
        return int(self.tile_keys.shape[0])

    @property
    def num_lower_nodes(self):
        return int(self.lower_origins.shape[0])

    @property
    def num_leaf_nodes(self):
        return int(self.leaf_origins.shape[0])

    @property
    def counts(self):
        return (self.num_upper_nodes, self.num_lower_nodes, self.num_leaf_nodes, self.num_voxels)

    @property
    def is_empty(self):
        return self.num_voxels == 0

    def __repr__(self):
        u, lo, f, v = self.counts
        label = f" {self.name!r}, " if self.name else ""
        return f"IndexGrid({label}upper={u}, lower={lo}, leaf={f}, voxels={v})"

    def leaf_occupancy(self):
        return 0.0 if self.num_leaf_nodes == 0 else self.num_voxels / (512.0 * self.num_leaf_nodes)

    def bbox(self):
        if self.is_empty:
            return None, None
        c = self.active_coords()
        return c.min(dim=0).values, c.max(dim=0).values

    def leaf_bbox(self):
        if self.is_empty:
            return None, None
        return self.leaf_origins.min(dim=0).values, self.leaf_origins.max(dim=0).values + (LEAF_SPAN - 1)

    # -- C-ABI view ----------------------------------------------------------
    def leaf_view(self) -> _lib.GridView:
        """GridView for kernels that read only the leaf arrays (a kernel map's OUTPUT grid): no node tables, so
        no table build (memsets + two kernels) for a grid that is never probed."""
        if self._view is not None:
            return self._view
        v = _lib.GridView()
        v.tile_keys = self.tile_keys.data_ptr()
        v.leaf_keys = self.leaf_keys.data_ptr()
        v.leaf_origins = self.leaf_origins.data_ptr()
        v.leaf_masks = self.leaf_masks.data_ptr()
        v.leaf_prefix = self.leaf_prefix.data_ptr()
        v.leaf_value_offset = self.leaf_value_offset.data_ptr()
        v.num_upper = self.num_upper_nodes
        v.num_leaf = self.num_leaf_nodes
        v.num_voxels = self.num_voxels
        return v

    def view(self) -> _lib.GridView:
        if self._view is None:
            v = _lib.GridView()
            v.tile_keys = self.tile_keys.data_ptr()
            v.leaf_keys = self.leaf_keys.data_ptr()
            v.leaf_origins = self.leaf_origins.data_ptr()
            v.leaf_masks = self.leaf_masks.data_ptr()
            v.leaf_prefix = self.leaf_prefix.data_ptr()
            v.leaf_value_offset = self.leaf_value_offset.data_ptr()
            v.num_upper = self.num_upper_nodes
            v.num_leaf = self.num_leaf_nodes
            v.num_voxels = self.num_voxels
            if self.num_leaf_nodes:  # dense child tables: probes become two loads after the tile search
                nu, nlo = self.num_upper_nodes, self.num_lower_nodes
                self._tables = (torch.empty(nu * 32768, dtype=torch.int32, device=self.device),
                                torch.empty(max(nlo, 1) * 4096, dtype=torch.int32, device=self.device))
                _lib.check(_lib.lib().fvdb_node_tables(
                    self.upper_child_starts.data_ptr(), nu, self.lower_offset_in_upper.data_ptr(),
                    self.lower_child_starts.data_ptr(), nlo, self.leaf_offset_in_lower.data_ptr(), self.num_leaf_nodes,
                    self._tables[0].data_ptr(), self._tables[1].data_ptr(), _lib.stream_ptr()), "node_tables")
                v.upper_table, v.lower_table = self._tables[0].data_ptr(), self._tables[1].data_ptr()
            self._view = v
        return self._view

    # -- queries (topology.py:253-299) ----------------------------------------
    def coord_to_index_many(self, coords):
        """1-based index per coordinate (0 = background), int64 CUDA tensor."""
        c = as_coords(coords, self.device)
        out = torch.empty(c.shape[0], dtype=torch.int64, device=self.device)
        if c.shape[0] == 0:
            return out
        L = _lib.lib()
        _lib.check(L.fvdb_coord_to_index(C.byref(self.view()), c.data_ptr(), c.shape[0], out.data_ptr(),
                                         _lib.stream_ptr()), "coord_to_index")
        return out

    def coord_to_index(self, i, j=None, k=None):
        if j is None:
            i, j, k = (int(x) for x in (i.as_tuple() if hasattr(i, "as_tuple") else i))
        return int(self.coord_to_index_many([[i, j, k]])[0].item())

    def active_coords(self):
        """[N,3] int64 coordinates in index order (row r has index r+1)."""
        out = torch.empty((self.num_voxels, 3), dtype=torch.int64, device=self.device)
        if self.num_voxels == 0:
            return out
        L = _lib.lib()
        _lib.check(L.fvdb_active_coords(C.byref(self.view()), out.data_ptr(), _lib.stream_ptr()),
                   "active_coords")
        return out

    # -- host export (parity / serialization) ------------------------------
    def to_numpy(self):
        """Dict of the topology arrays with the reference's numpy dtypes (bit-exact)."""
        out = {}
        for f in ARRAY_FIELDS:
            a = getattr(self, f).cpu().numpy()
            out[f] = a.view(_NP_DTYPES[f]) if a.dtype.itemsize == np.dtype(_NP_DTYPES[f]).itemsize else a
        out["num_voxels"] = self.num_voxels
        return out


def as_coords(coords, device) -> torch.Tensor:
    """[N,3] int64 contiguous CUDA tensor from array-likes (reshape(-1,3) like the reference)."""
    if isinstance(coords, torch.Tensor):
        t = coords.to(device=device, dtype=torch.int64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(coords, np.int64))).to(device)
    return t.reshape(-1, 3).contiguous()


def empty_grid(transform=None, name="", device=None):
    """A grid with no active voxels (topology.py:386-404)."""
    dev = device or _device()
    z = {f: torch.zeros((0,), dtype=_TORCH_DTYPES[f], device=dev) for f in ARRAY_FIELDS}
    for f in ("upper_origins", "lower_origins", "leaf_origins"):
        z[f] = torch.zeros((0, 3), dtype=torch.int64, device=dev)
    z["leaf_masks"] = torch.zeros((0, 8), dtype=torch.int64, device=dev)
    z["upper_child_starts"] = torch.zeros(1, dtype=torch.int64, device=dev)
    z["lower_child_starts"] = torch.zeros(1, dtype=torch.int64, device=dev)
    return IndexGrid(num_voxels=0, transform=transform or VoxelTransform.uniform(1.0), name=name, **z)
