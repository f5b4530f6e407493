"""Order-sensitive digests of full-size grids and kernel maps (shared by the golden generator and the tests).

A digest is SHA-256 over the array's bytes in the reference's dtype and C order, so it pins every value AND
its position: the active-voxel ordering, the node order and the per-offset pair order (out_rows ascending,
conv.py:87).  Kernel map: one SHA-256 over in_rows[0] ‖ … ‖ in_rows[26] ‖ out_rows[0] ‖ … ‖ out_rows[26],
each int64 little-endian (the reference's KernelMap lists, conv.py:80-122).
"""
from __future__ import annotations

import hashlib

import numpy as np

FIELDS = ("tile_keys", "upper_origins", "upper_child_starts", "lower_offset_in_upper", "lower_origins",
          "lower_child_starts", "leaf_offset_in_lower", "leaf_keys", "leaf_origins", "leaf_masks",
          "leaf_prefix", "leaf_value_offset")


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype.byteorder == ">":
        a = a.astype(a.dtype.newbyteorder("<"))
    return hashlib.sha256(a.tobytes()).hexdigest()


def grid_digest(arrays: dict, active_coords, counts) -> dict:
    d = {f: sha(arrays[f]) for f in FIELDS}
    d["active_coords"] = sha(np.asarray(active_coords, dtype=np.int64))
    d["counts"] = [int(c) for c in counts]
    return d


def map_digest(chunks_in, chunks_out, counts) -> dict:
    """chunks_*: iterables of int64 arrays (the 27 per-offset lists, in offset order)."""
    h = hashlib.sha256()
    for a in chunks_in:
        h.update(np.ascontiguousarray(np.asarray(a, dtype="<i8")).tobytes())
    for a in chunks_out:
        h.update(np.ascontiguousarray(np.asarray(a, dtype="<i8")).tobytes())
    return {"pairs_sha256": h.hexdigest(), "pair_counts": [int(c) for c in counts], "total_pairs": int(sum(counts))}
