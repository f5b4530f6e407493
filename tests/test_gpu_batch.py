"""GPU parity: batched (jagged) grid build and batched kernel map.

Every element of a batched build must be bit-identical to its standalone build, which the reference-golden
tests (test_gpu_grid.py) pin to the reference itself; the reference assembles a GridBatch from per-element
builds (jagged.py:112-123) and conv_batch runs per element (conv.py:371-383), so the batched kernel map must
equal the per-element maps concatenated with row offsets.
"""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import lidar_scan_points, random_points, sphere_shell_coords
from conftest import FIELDS, GRID_CASES

pytestmark = pytest.mark.gpu


def _arrays_equal(a, b):
    x, y = a.to_numpy(), b.to_numpy()
    for f in FIELDS:
        assert x[f].dtype == y[f].dtype and x[f].shape == y[f].shape, f
        assert np.array_equal(x[f], y[f]), f
    assert a.num_voxels == b.num_voxels


def _jag(arrs):
    return P.jagged_from_list([torch.as_tensor(np.ascontiguousarray(a)) for a in arrs])


def _mixed_elements(golden_grids):
    return [golden_grids[f"{n}/coords"] for n in GRID_CASES]


def test_batched_build_equals_standalone(golden_grids):
    elems = _mixed_elements(golden_grids)  # one root tile, several tiles, +-2^30 extremes, duplicates
    batch, stats = P.build_from_coords(_jag(elems))
    assert isinstance(batch, P.GridBatch) and batch.num_grids == len(elems)
    for b, c in enumerate(elems):
        g, _ = P.build_from_coords(c)
        _arrays_equal(batch.grids[b], g)
        og = O.build_from_coords(c)  # and the oracle restatement (pinned to the reference goldens)
        a = batch.grids[b].to_numpy()
        for f in FIELDS:
            assert np.array_equal(a[f], getattr(og, f)), (b, f)
    assert stats.unique_count == batch.total_voxels


def test_batched_build_single_sort_path(golden_grids):
    """Elements whose tile keys fit the batched sort key (no +-2^30 extremes): the one-pass path proper."""
    names = [n for n in GRID_CASES if n != "wide"]
    elems = [golden_grids[f"{n}/coords"] for n in names]
    batch, stats = P.build_from_coords(_jag(elems))
    assert "plan" in stats.phase_seconds  # not the element-by-element fallback
    for b, n in enumerate(names):
        a = batch.grids[b].to_numpy()
        for f in FIELDS:
            assert np.array_equal(a[f], golden_grids[f"{n}/{f}"]), (n, f)


def test_batched_build_shared_tile_and_empty_elements():
    rng = np.random.default_rng(3)
    elems = [rng.integers(-40, 40, size=(n, 3)) for n in (500, 0, 1, 2000, 0)]
    batch, _ = P.build_batch_from_coords(_jag(elems))
    for b, c in enumerate(elems):
        g, _ = P.build_from_coords(c)
        assert batch.grids[b].num_voxels == g.num_voxels
        if c.shape[0]:
            _arrays_equal(batch.grids[b], g)
    assert batch.voxel_joffsets[:, 1].tolist() == np.cumsum([batch.grids[b].num_voxels
                                                             for b in range(5)]).tolist()


def test_batched_points_equals_standalone():
    pts = [lidar_scan_points(s)[::7] for s in range(3)] + [random_points(np.random.default_rng(0), 5000, 1.0)]
    tf = P.VoxelTransform.uniform(0.05)
    batch, _ = P.build_from_points(_jag(pts), tf)
    for b, p in enumerate(pts):
        g, _ = P.build_from_points(p, tf)
        _arrays_equal(batch.grids[b], g)


def test_batched_build_errors_name_the_row():
    good = np.zeros((4, 3), np.int64)
    bad = np.array([[0, 0, 0], [0, (1 << 30) + 1, 0]], np.int64)
    with pytest.raises(ValueError, match=r"coordinate out of range at row 5: \(0, 1073741825, 0\)"):
        P.build_from_coords(_jag([good, bad]))
    pts = np.zeros((3, 3))
    pts[2, 1] = np.nan
    with pytest.raises(ValueError, match=r"non-finite point at row 6"):
        P.build_from_points(_jag([np.ones((4, 3)), pts]), P.VoxelTransform.uniform(1.0))


def _concat_maps(gi, go, stride):
    """Reference semantics: per-element maps with batch row offsets (conv.py:371-383)."""
    tabs, counts, oi, oo = [], np.zeros(27, np.int64), 0, 0
    for a, b in zip(gi, go):
        km = P.build_kernel_map(a, b, stride)
        t = km.nbr.cpu().numpy().astype(np.int64)
        tabs.append(np.where(t >= 0, t + oi, -1))
        counts += km.pair_counts
        oi += a.num_voxels
        oo += b.num_voxels
    return np.concatenate(tabs, 1), counts


@pytest.mark.parametrize("stride", [1, 2])
def test_batched_kernel_map_equals_per_element(stride):
    pts = [lidar_scan_points(s)[::5] for s in range(4)]
    fine, _ = P.build_from_points(_jag(pts), P.VoxelTransform.uniform(0.05))
    out = fine if stride == 1 else P.coarsen_batch(fine, 2)
    for b in range(fine.num_grids):  # batched coarsen == standalone coarsen
        if stride == 2:
            _arrays_equal(out.grids[b], P.coarsen(fine.grids[b], 2))
    km = P.build_batch_kernel_map(fine, out, stride)
    ref, counts = _concat_maps(fine.grids, out.grids, stride)
    assert np.array_equal(km.nbr.cpu().numpy(), ref)
    assert np.array_equal(km.pair_counts, counts)
    assert (km.fwd.t[:, km.num_out:] == -1).all()


def test_batched_kernel_map_many_elements():
    """More elements than one launch chunk (32) and separately built (non-contiguous) grids."""
    rng = np.random.default_rng(5)
    grids = [P.build_from_coords(rng.integers(-30, 30, size=(int(rng.integers(1, 400)), 3)))[0] for _ in range(37)]
    batch = P.GridBatch(grids)
    km = P.build_batch_kernel_map(batch, batch, 1)
    ref, counts = _concat_maps(grids, grids, 1)
    assert np.array_equal(km.nbr.cpu().numpy(), ref)
    assert np.array_equal(km.pair_counts, counts)


def test_conv_batch_on_batched_build_equals_per_element():
    pts = [lidar_scan_points(s)[::9] for s in range(3)]
    batch, _ = P.build_from_points(_jag(pts), P.VoxelTransform.uniform(0.05))
    rng = np.random.default_rng(1)
    x = torch.from_numpy(rng.normal(size=(batch.total_voxels, 16)).astype(np.float32)).cuda()
    w = torch.from_numpy((rng.normal(size=(8, 16, 3, 3, 3)) / np.sqrt(27 * 16)).astype(np.float32))
    y = P.conv_batch(batch, batch.jagged(x), w).jdata
    for b, g in enumerate(batch.grids):
        sl = batch.voxel_slice(b)
        yb = P.conv(g, x[sl], w)
        assert torch.equal(y[sl], yb)


def test_sparse_conv_module_on_bare_grid_reuses_maps():
    g, _ = P.build_from_coords(sphere_shell_coords(40, band=1.5))
    m = P.SparseConv3d(32, 32).cuda()
    x = torch.randn(g.num_voxels, 32, device="cuda")
    m(g, x)
    m(g, x)
    from paper_2407_01781_b200.conv import cached_batch_kernel_map
    km = cached_batch_kernel_map(P.as_grid_batch(g), P.as_grid_batch(g), 1)
    assert km is not None and km.fwd.uses == 2
