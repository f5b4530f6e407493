"""``FVDBIDX1`` grid files (drop-in for reference ``idxgrid.io`` save_grid / load_grid, io.py:1-180).

Byte-identical to the reference writer (same layout, same record order, little-endian, no padding):

    magic "FVDBIDX1" | version u32 | counts 4 x u64 | xform 6 x f64 | name u32 + utf-8
    upper records:  tile_key u64, child_count u32, child offsets u16 x count
    lower records:  child_count u32, child offsets u16 x count
    leaf records:   value_offset u64, prefix u64, mask 8 x u64    (80 bytes)

The 80-byte leaf records are exactly the device leaf arrays (value offsets, prefixes, masks), so a
load is one upload of the record block plus a top-down origin/key reconstruction; the variable-length
internal records are (de)serialised with vectorised numpy instead of the reference's per-record loop.
Errors are :class:`GridFileError` (a ``ValueError``) with the reference's messages.
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from .topology import ARRAY_FIELDS, IndexGrid, VoxelTransform, _TORCH_DTYPES, _device, empty_grid

MAGIC = b"FVDBIDX1"
VERSION = 1
LEAF_RECORD_BYTES = 80
_HEADER = struct.Struct("<8sI4Q6dI")


class GridFileError(ValueError):
    """Raised for malformed grid files (bad magic, version, or truncation) (io.py:36-37)."""


def _records(heads: np.ndarray, counts: np.ndarray, children: np.ndarray) -> bytes:
    """Concatenate variable-length records: head bytes of each node, then its u16 child offsets."""
    n = len(counts)
    if n == 0:
        return b""
    hb = heads.shape[1]
    sizes = hb + 2 * counts.astype(np.int64)
    starts = np.concatenate(([0], np.cumsum(sizes)[:-1]))
    out = np.zeros(int(sizes.sum()), np.uint8)
    out[(starts[:, None] + np.arange(hb)[None, :]).ravel()] = heads.ravel()
    cb = children.astype("<u2").view(np.uint8)
    first = np.concatenate(([0], np.cumsum(counts)[:-1])).astype(np.int64)  # first child of each node
    child_node = np.repeat(np.arange(n), counts)
    pos = starts[child_node] + hb + 2 * (np.arange(len(children)) - first[child_node])
    out[(pos[:, None] + np.arange(2)[None, :]).ravel()] = cb
    return out.tobytes()


def save_grid(grid, path):
    """Write a grid; returns the byte count.  Output bytes equal the reference writer's (io.py:40-70)."""
    a = grid.to_numpy()
    name = grid.name.encode("utf-8")
    t = grid.transform
    parts = [_HEADER.pack(MAGIC, VERSION, *(int(c) for c in grid.counts), *np.asarray(t.voxel_size, np.float64),
                          *np.asarray(t.origin, np.float64), len(name)), name]
    ucs = a["upper_child_starts"].astype(np.int64)
    nu = len(a["tile_keys"])
    if nu:
        heads = np.zeros((nu, 12), np.uint8)
        heads[:, :8] = a["tile_keys"].astype("<u8").view(np.uint8).reshape(nu, 8)
        heads[:, 8:] = np.diff(ucs).astype("<u4").view(np.uint8).reshape(nu, 4)
        parts.append(_records(heads, np.diff(ucs), a["lower_offset_in_upper"]))
    lcs = a["lower_child_starts"].astype(np.int64)
    nl = len(lcs) - 1 if len(lcs) else 0
    if nl > 0:
        heads = np.diff(lcs).astype("<u4").view(np.uint8).reshape(nl, 4)
        parts.append(_records(heads, np.diff(lcs), a["leaf_offset_in_lower"]))
    nf = len(a["leaf_value_offset"])
    leaf = np.empty((nf, 10), dtype="<u8")
    leaf[:, 0] = a["leaf_value_offset"]
    leaf[:, 1] = a["leaf_prefix"]
    leaf[:, 2:] = a["leaf_masks"]
    parts.append(leaf.tobytes())
    blob = b"".join(parts)
    with open(path, "wb") as fh:
        fh.write(blob)
    return len(blob)


def _parse_records(blob: memoryview, pos: int, n: int, head: int, what: str):
    """Walk n variable-length records (head bytes whose last 4 are the u32 child count) from pos."""
    counts = np.empty(n, np.int64)
    starts = np.empty(n, np.int64)
    total = len(blob)
    for i in range(n):
        if pos + head > total:
            raise GridFileError(f"truncated grid file: needed {head} bytes for {what} record {i} at offset "
                                f"{pos}, have {total - pos}")
        (cnt,) = struct.unpack_from("<I", blob, pos + head - 4)
        starts[i] = pos
        counts[i] = cnt
        pos += head
        if pos + 2 * cnt > total:
            raise GridFileError(f"truncated grid file: needed {2 * cnt} bytes for {what} {i} children at offset "
                                f"{pos}, have {total - pos}")
        pos += 2 * cnt
    return counts, starts, pos


def load_grid(path, device=None):
    """Read a grid written by :func:`save_grid` or the reference (io.py:88-180) onto the device."""
    with open(path, "rb") as fh:
        raw = fh.read()
    blob = memoryview(raw)
    if len(raw) < _HEADER.size:
        raise GridFileError(f"truncated grid file: needed {_HEADER.size} bytes for header at offset 0, "
                            f"have {len(raw)}")
    magic, version, nu, nl, nf, nv, *rest = _HEADER.unpack_from(raw, 0)
    if magic != MAGIC:
        raise GridFileError(f"bad magic at offset 0: expected {MAGIC!r}, got {bytes(magic)!r}")
    if version != VERSION:
        raise GridFileError(f"unsupported grid file version {version} (expected {VERSION})")
    vs, og, name_len = rest[0:3], rest[3:6], rest[6]
    pos = _HEADER.size
    if pos + name_len > len(raw):
        raise GridFileError(f"truncated grid file: needed {name_len} bytes for name at offset {pos}, "
                            f"have {len(raw) - pos}")
    name = bytes(blob[pos:pos + name_len]).decode("utf-8")
    pos += name_len
    transform = VoxelTransform(np.array(vs), np.array(og))
    dev = device or _device()
    if nf == 0:
        return empty_grid(transform, name, device=dev)
    u8 = np.frombuffer(raw, np.uint8)

    def children(counts, starts, head):
        idx = np.repeat(starts + head, counts) + 2 * (np.arange(int(counts.sum())) -
                                                      np.repeat(np.concatenate(([0], np.cumsum(counts)[:-1])), counts))
        b = u8[(idx[:, None] + np.arange(2)[None, :]).ravel()]
        return b.view("<u2").astype(np.uint16)

    ucnt, ust, pos = _parse_records(blob, pos, nu, 12, "upper")
    tile_keys = np.array([struct.unpack_from("<Q", raw, int(s))[0] for s in ust], np.uint64)
    lower_offset_in_upper = children(ucnt, ust, 12) if nu else np.zeros(0, np.uint16)
    if len(lower_offset_in_upper) != nl:
        raise GridFileError(f"lower node count mismatch: header says {nl}, records hold "
                            f"{len(lower_offset_in_upper)}")
    lcnt, lst, pos = _parse_records(blob, pos, nl, 4, "lower")
    leaf_offset_in_lower = children(lcnt, lst, 4) if nl else np.zeros(0, np.uint16)
    if len(leaf_offset_in_lower) != nf:
        raise GridFileError(f"leaf count mismatch: header says {nf}, records hold {len(leaf_offset_in_lower)}")
    need = nf * LEAF_RECORD_BYTES
    if pos + need > len(raw):
        raise GridFileError(f"truncated grid file: needed {need} bytes for leaf records at offset {pos}, "
                            f"have {len(raw) - pos}")
    leaf = np.frombuffer(raw, "<u8", count=nf * 10, offset=pos).reshape(nf, 10)
    pos += need
    if pos != len(raw):
        raise GridFileError(f"{len(raw) - pos} trailing bytes after leaf records")

    # origins and leaf keys, top-down from the tile keys and local offsets (io.py:142-162)
    f = ((tile_keys[:, None] >> np.array([42, 21, 0], np.uint64)) & np.uint64(0x1FFFFF)).astype(np.int64)
    upper_origins = (((f + (1 << 20)) & 0x1FFFFF) - (1 << 20)) << 12
    upper_starts = np.concatenate(([0], np.cumsum(ucnt))).astype(np.int64)
    upper_of_lower = np.repeat(np.arange(nu), ucnt)
    ul = lower_offset_in_upper.astype(np.int64)
    lower_origins = upper_origins[upper_of_lower] + np.stack(
        [((ul >> 10) & 31) << 7, ((ul >> 5) & 31) << 7, (ul & 31) << 7], 1)
    lower_starts = np.concatenate(([0], np.cumsum(lcnt))).astype(np.int64)
    lower_of_leaf = np.repeat(np.arange(nl), lcnt)
    ll = leaf_offset_in_lower.astype(np.int64)
    leaf_origins = lower_origins[lower_of_leaf] + np.stack(
        [((ll >> 8) & 15) << 3, ((ll >> 4) & 15) << 3, (ll & 15) << 3], 1)
    leaf_keys = ((upper_of_lower[lower_of_leaf].astype(np.uint64) << np.uint64(27))
                 | (ul[lower_of_leaf].astype(np.uint64) << np.uint64(12)) | ll.astype(np.uint64))
    pops = int(np.bitwise_count(leaf[:, 2:]).sum())
    if pops != nv:
        raise GridFileError(f"active voxel count mismatch: header {nv}, masks {pops}")

    rec = torch.from_numpy(leaf.view(np.int64).copy()).to(dev)  # the leaf records are the device leaf arrays
    host = {"tile_keys": tile_keys, "upper_origins": upper_origins, "upper_child_starts": upper_starts,
            "lower_offset_in_upper": lower_offset_in_upper, "lower_origins": lower_origins,
            "lower_child_starts": lower_starts, "leaf_offset_in_lower": leaf_offset_in_lower,
            "leaf_keys": leaf_keys, "leaf_origins": leaf_origins}
    arrays = {}
    for k, v in host.items():
        v = np.ascontiguousarray(v)
        arrays[k] = torch.from_numpy(v.view(np.int16) if v.dtype == np.uint16 else v.view(np.int64)).to(dev)
    arrays["leaf_value_offset"] = rec[:, 0].contiguous()
    arrays["leaf_prefix"] = rec[:, 1].contiguous()
    arrays["leaf_masks"] = rec[:, 2:].contiguous()
    assert set(arrays) == set(ARRAY_FIELDS) and all(arrays[k].dtype == _TORCH_DTYPES[k] for k in arrays)
    return IndexGrid(num_voxels=int(nv), transform=transform, name=name, **arrays)
