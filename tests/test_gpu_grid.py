"""GPU parity: index-grid build, probes and kernel maps are bit-exact vs the reference goldens."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import lidar_scan_points, random_points, sphere_shell_coords
from conftest import FIELDS, GRID_CASES, KMAP_CASES

pytestmark = pytest.mark.gpu


def assert_grid_equal(g, golden, prefix):
    a = g.to_numpy()
    for f in FIELDS:
        ref = golden[f"{prefix}/{f}"]
        assert a[f].dtype == ref.dtype, (f, a[f].dtype, ref.dtype)
        assert a[f].shape == ref.shape, (f, a[f].shape, ref.shape)
        assert np.array_equal(a[f], ref), f
    assert g.num_voxels == int(golden[f"{prefix}/num_voxels"])


@pytest.mark.parametrize("name", GRID_CASES)
def test_build_bit_exact(golden_grids, name):
    g, stats = P.build_from_coords(golden_grids[f"{name}/coords"])
    assert_grid_equal(g, golden_grids, name)
    assert stats.unique_count == g.num_voxels and stats.num_leaf == g.num_leaf_nodes
    assert np.array_equal(g.active_coords().cpu().numpy(), golden_grids[f"{name}/active_coords"])
    idx = g.coord_to_index_many(golden_grids[f"{name}/probe"]).cpu().numpy()
    assert np.array_equal(idx, golden_grids[f"{name}/probe_index"])
    assert_grid_equal(P.coarsen(g, 2), golden_grids, f"{name}/coarse2")


@pytest.mark.parametrize("name", ["scattered", "multi_tile", "wide", "dup_heavy"])
def test_build_permutation_invariant(golden_grids, name):
    c = golden_grids[f"{name}/coords"]
    perm = np.random.default_rng(0).permutation(len(c))
    g, _ = P.build_from_coords(np.concatenate([c[perm], c[:7]]))
    assert_grid_equal(g, golden_grids, name)


def test_points_path_bit_exact(golden_grids):
    p = golden_grids["points/points"]
    t = P.VoxelTransform(golden_grids["points/voxel_size"], golden_grids["points/origin"])
    assert np.array_equal(t.quantize(p).cpu().numpy(), golden_grids["points/quantized"])
    g, _ = P.build_from_points(p, t)
    assert_grid_equal(g, golden_grids, "points")


def test_reference_frontend_fixtures(golden_fixtures):
    fx = golden_fixtures
    g, _ = P.build_from_points(fx["points"], P.VoxelTransform(fx["voxel_size"], fx["origin"]))
    assert list(g.counts) == fx["counts"].tolist()
    assert np.array_equal(g.active_coords().cpu().numpy(), fx["active_coords"])
    assert np.array_equal(g.coord_to_index_many(fx["probe_coords"]).cpu().numpy(), fx["probe_expected"])


def test_build_errors_match_reference_text():
    with pytest.raises(ValueError, match=r"coordinate out of range at row 1: \(0, 1073741825, 0\) "
                                         r"\(components must be within \+-1073741824\)"):
        P.build_from_coords([[0, 0, 0], [0, (1 << 30) + 1, 0], [0, 0, -(1 << 31)]])
    with pytest.raises(ValueError, match=r"non-finite point at row 2: \[nan, 0.0, 0.0\]"):
        P.build_from_points([[0, 0, 0], [1, 1, 1], [np.nan, 0, 0]], P.VoxelTransform.uniform(1.0))
    g, st = P.build_from_coords(np.zeros((0, 3), np.int64))
    assert g.counts == (0, 0, 0, 0) and st.input_count == 0
    assert g.coord_to_index_many([[0, 0, 0]]).tolist() == [0]


def test_build_from_points_reports_nonfinite_before_range():
    """The finite check is deferred into the build's first read-back: it must still win over the range
    check (the reference quantizes, raising on non-finite points, before it builds)."""
    pts = [[1e12, 0.0, 0.0], [0.0, 0.0, 0.0], [0.0, np.inf, 0.0]]
    with pytest.raises(ValueError, match=r"non-finite point at row 2: \[0.0, inf, 0.0\]"):
        P.build_from_points(pts, P.VoxelTransform.uniform(1.0))
    with pytest.raises(ValueError, match=r"coordinate out of range at row 0"):
        P.build_from_points(pts[:2], P.VoxelTransform.uniform(1.0))


def test_build_from_points_with_many_duplicates():
    """Node scans run over all input slots with the tail past the unique count masked: a cloud that
    collapses ~7:1 onto voxels must give the oracle's grid exactly."""
    rng = np.random.default_rng(11)
    pts = rng.normal(size=(50_000, 3)) * 4.0
    g, st = P.build_from_points(pts, P.VoxelTransform.uniform(1.0))
    og = O.build_from_points(pts, (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    assert g.num_voxels < 10_000 and st.input_count == 50_000 and g.num_voxels == og.num_voxels
    a = g.to_numpy()
    for f in FIELDS:
        assert np.array_equal(a[f], getattr(og, f)), f


def test_coord_limit_edge_is_accepted():
    c = np.array([[1 << 30, -(1 << 30), 0], [-(1 << 30), 1 << 30, (1 << 30)]])
    g, _ = P.build_from_coords(c)
    og = O.build_from_coords(c)
    a = g.to_numpy()
    for f in FIELDS:
        assert np.array_equal(a[f], getattr(og, f)), f


@pytest.mark.parametrize("name", KMAP_CASES)
@pytest.mark.parametrize("stride", [1, 2])
def test_kernel_map_bit_exact(golden_grids, golden_kmaps, name, stride):
    g, _ = P.build_from_coords(golden_grids[f"{name}/coords"])
    go = g if stride == 1 else P.coarsen(g, 2)
    km = P.build_kernel_map(g, go, stride)
    key = f"{name}/s{stride}"
    assert np.array_equal(km.pair_counts, golden_kmaps[f"{key}/counts"])
    assert np.array_equal(torch.cat(km.in_rows).cpu().numpy(), golden_kmaps[f"{key}/in_rows"])
    assert np.array_equal(torch.cat(km.out_rows).cpu().numpy(), golden_kmaps[f"{key}/out_rows"])
    assert km.num_in == g.num_voxels and km.num_out == go.num_voxels and km.stride == stride


def test_kernel_map_known_answers():
    g, _ = P.build_from_coords([(0, 0, 0)])
    km = P.build_kernel_map(g, g, 1)
    assert km.pair_counts[P.KernelMap.offset_index(0, 0, 0)] == 1 and km.total_pairs == 1
    g, _ = P.build_from_coords([(0, 0, 0), (1, 0, 0)])
    c = P.build_kernel_map(g, g, 1).pair_counts
    assert c[13] == 2 and c[P.KernelMap.offset_index(1, 0, 0)] == 1 and c[P.KernelMap.offset_index(-1, 0, 0)] == 1
    assert c.sum() == 4


def test_kernel_map_across_grids_and_empty():
    rng = np.random.default_rng(4)
    a = rng.integers(-20, 20, size=(500, 3))
    b = rng.integers(-20, 20, size=(300, 3))
    ga, gb = P.build_from_coords(a)[0], P.build_from_coords(b)[0]
    km = P.build_kernel_map(ga, gb, 1)
    ins, outs = O.kernel_map(O.build_from_coords(a), O.build_from_coords(b), 1)
    assert np.array_equal(torch.cat(km.in_rows).cpu().numpy(), np.concatenate(ins))
    assert np.array_equal(torch.cat(km.out_rows).cpu().numpy(), np.concatenate(outs))
    e = P.empty_grid()
    assert P.build_kernel_map(e, ga, 1).total_pairs == 0
    assert P.build_kernel_map(ga, e, 1).total_pairs == 0


def test_transposed_table_is_inverse():
    rng = np.random.default_rng(5)
    g, _ = P.build_from_coords(rng.integers(-30, 30, size=(4000, 3)))
    g2 = P.coarsen(g, 2)
    for gi, go, s in ((g, g, 1), (g, g2, 2)):
        km = P.build_kernel_map(gi, go, s)
        t = km.transposed_table().cpu().numpy()
        nbr = km.nbr.cpu().numpy()
        for d in range(27):
            o = np.flatnonzero(nbr[d] >= 0)
            assert np.array_equal(t[d][nbr[d][o]], o)
            assert (t[d] >= 0).sum() == len(o)
        if s == 1:  # offset symmetry d <-> -d (reference test_conv.py:80-89)
            assert np.array_equal(t, nbr[::-1])


@pytest.mark.slow
def test_cfg1_points_counts(golden_sizes):
    pts = random_points(np.random.default_rng(0), 100_000, sigma=1.0)
    g, _ = P.build_from_points(pts, P.VoxelTransform.uniform(0.05))
    assert list(g.counts) == golden_sizes["cfg1"]["counts"]
    km = P.build_kernel_map(g, g, 1)
    assert km.total_pairs == golden_sizes["cfg1"]["pairs"]
    assert km.pair_counts.tolist() == golden_sizes["cfg1"]["pair_counts"]


@pytest.mark.slow
def test_cfg2_full_size_bit_exact_counts(golden_sizes):
    c = sphere_shell_coords(470, band=1.5)
    g, _ = P.build_from_coords(c)
    ref = golden_sizes["cfg2"]
    assert list(g.counts) == ref["counts"]
    ac = g.active_coords().cpu().numpy()
    assert int((ac * np.array([1, 7919, 104729])).sum() % (1 << 61)) == ref["coord_checksum"]
    km = P.build_kernel_map(g, g, 1)
    assert km.total_pairs == ref["pairs"] and km.pair_counts.tolist() == ref["pair_counts"]
    # every output's neighbour at offset d really is coord+δ_d (probe via the independent path)
    nbr = km.nbr
    rows = torch.arange(0, g.num_voxels, 997, device=nbr.device)
    acd = g.active_coords()
    for d in (0, 4, 13, 22, 26):
        q = acd[rows] + torch.tensor(P.STENCIL[d], device=nbr.device)
        idx = g.coord_to_index_many(q) - 1
        assert torch.equal(idx.to(torch.int32), nbr[d, rows])
    g2 = P.coarsen(g, 2)
    assert list(g2.counts) == golden_sizes["cfg4"]["coarse_counts"]
    k2 = P.build_kernel_map(g, g2, 2)
    assert k2.total_pairs == golden_sizes["cfg4"]["pairs_s2"]
    assert k2.pair_counts.tolist() == golden_sizes["cfg4"]["pair_counts_s2"]


@pytest.mark.slow
def test_cfg3_lidar_counts(golden_sizes):
    for ref in golden_sizes["cfg3"]:
        g, _ = P.build_from_points(lidar_scan_points(ref["seed"]), P.VoxelTransform.uniform(0.05))
        assert list(g.counts) == ref["counts"]
        assert P.build_kernel_map(g, g, 1).total_pairs == ref["pairs"]


@pytest.mark.parametrize("name", KMAP_CASES)
def test_same_grid_transpose_by_row_reversal_is_exact(golden_grids, name):
    """Stride-1 maps of a grid onto itself build the transposed table by reversing the offset rows
    (nbr[d][o] = i <=> nbr[26-d][i] = o): bit-identical to the scatter transpose (fvdb_kmap_transpose)."""
    from paper_2407_01781_b200 import _lib
    from paper_2407_01781_b200.conv import padded_len
    key = f"{name}/active_coords"
    if key not in golden_grids:
        pytest.skip("no coordinates in this golden case")
    c = golden_grids[key]
    g, _ = P.build_from_coords(c)
    km = P.build_kernel_map(g, g, 1)
    t = torch.empty((27, padded_len(g.num_voxels)), dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().fvdb_kmap_transpose(km.fwd.t.data_ptr(), km.fwd.ld, km.num_out, km.num_in, t.data_ptr(),
                                              t.shape[1], _lib.stream_ptr()), "kmap_transpose")
    assert km._same_grids() and torch.equal(km.bwd.t, t)


@pytest.mark.parametrize("name", ["multi_tile", "neg_boundary", "scattered", "wide"])
def test_probe_with_and_without_node_tables(golden_grids, name):
    """coord_to_index through the dense child tables (default views) equals the binary-search path (a view without
    tables) and the reference's probe results."""
    import ctypes as C
    from paper_2407_01781_b200 import _lib
    g, _ = P.build_from_coords(golden_grids[f"{name}/coords"])
    q = torch.from_numpy(np.ascontiguousarray(golden_grids[f"{name}/probe"])).cuda()
    with_t = g.coord_to_index_many(q)
    v = g.view()
    assert v.lower_table
    bare = _lib.GridView(tile_keys=v.tile_keys, leaf_keys=v.leaf_keys, leaf_origins=v.leaf_origins,
                         leaf_masks=v.leaf_masks, leaf_prefix=v.leaf_prefix, leaf_value_offset=v.leaf_value_offset,
                         num_upper=v.num_upper, num_leaf=v.num_leaf, num_voxels=v.num_voxels)
    out = torch.empty(q.shape[0], dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().fvdb_coord_to_index(C.byref(bare), q.data_ptr(), q.shape[0], out.data_ptr(),
                                              _lib.stream_ptr()), "coord_to_index")
    assert torch.equal(with_t, out)
    assert np.array_equal(with_t.cpu().numpy(), golden_grids[f"{name}/probe_index"])


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_coarsen2_from_leaves_matches_coordinate_build(seed):
    """coarsen(g, 2) runs from the fine leaves (fvdb_coarsen2_*); it must equal the coordinate build of
    unique(ijk // 2) in every array, including negative coordinates (arithmetic floor) and sparse / dense mixes."""
    from paper_2407_01781_b200.build import _coarsen2_leaves
    rng = np.random.default_rng(seed)
    c = np.concatenate([rng.integers(-300, 300, size=(20000, 3)),
                        sphere_shell_coords(60, band=1.5) - 40,
                        rng.integers(-9, 9, size=(3000, 3))])
    # one root tile (negative coordinates: tile -1) for the leaf path; the multi-tile input falls back
    multi, _ = P.build_from_coords(c)
    assert _coarsen2_leaves(multi, multi.transform) is None
    g, _ = P.build_from_coords(c - 2000)
    fast = _coarsen2_leaves(g, g.transform)
    assert fast is not None
    ref, _ = P.build_from_coords(np.floor_divide(g.active_coords().cpu().numpy(), 2))
    a, b = fast.to_numpy(), ref.to_numpy()
    for f in FIELDS:
        assert a[f].dtype == b[f].dtype and np.array_equal(a[f], b[f]), f
    assert fast.num_voxels == ref.num_voxels


@pytest.mark.parametrize("seed", [0, 1])
def test_leaf_hash_build_matches_coordinate_build(seed):
    """The leaf-hash build (default for one root tile) against the coordinate build (FVDB_BUILD_LEAF=0 path):
    duplicates, negative coordinates, dense and scattered parts; and its fallback on a multi-tile input."""
    from paper_2407_01781_b200 import build as B
    rng = np.random.default_rng(seed)
    # ~3.6K leaves for ~38K voxels: under half of the n / 4 table entries (a crowded table falls back, below)
    c = np.concatenate([rng.integers(-2400, -1700, size=(2000, 3)), sphere_shell_coords(80, band=1.5) - 2000,
                        rng.integers(-2100, -2090, size=(5000, 3))])
    c = np.concatenate([c, c[:777]])  # duplicates
    cc = torch.from_numpy(c).cuda()
    fast = B._build_leaf(cc, P.VoxelTransform.uniform(1.0), "", B.BuildStats())
    assert fast is not None
    try:
        B._LEAF_BUILD = False
        ref, _ = P.build_from_coords(c)
    finally:
        B._LEAF_BUILD = True
    a, b = fast.to_numpy(), ref.to_numpy()
    for f in FIELDS:
        assert a[f].dtype == b[f].dtype and np.array_equal(a[f], b[f]), f
    assert fast.num_voxels == ref.num_voxels
    multi = torch.from_numpy(rng.integers(-5000, 5000, size=(1000, 3))).cuda()  # several root tiles
    assert B._build_leaf(multi, P.VoxelTransform.uniform(1.0), "", B.BuildStats()) is None
    crowded = torch.from_numpy(rng.integers(0, 4000, size=(20000, 3))).cuda()  # ~1 voxel per leaf
    assert B._build_leaf(crowded, P.VoxelTransform.uniform(1.0), "", B.BuildStats()) is None
    g, _ = P.build_from_coords(crowded)  # falls back to the coordinate build
    assert g.num_voxels == len(np.unique(crowded.cpu().numpy(), axis=0))
