"""CPU: the oracle (numpy restatement) reproduces the reference's golden vectors bit-exactly."""
import numpy as np
import pytest

import oracle as O
from conftest import CONV_CASES, FIELDS, GRID_CASES, KMAP_CASES


def _grid(gg, name):
    return O.build_from_coords(gg[f"{name}/coords"])


@pytest.mark.parametrize("name", GRID_CASES)
def test_oracle_grid_arrays_match_reference(golden_grids, name):
    g = _grid(golden_grids, name)
    for f in FIELDS:
        ref = golden_grids[f"{name}/{f}"]
        got = getattr(g, f)
        assert got.dtype == ref.dtype, f
        assert np.array_equal(got, ref), f
    assert g.num_voxels == int(golden_grids[f"{name}/num_voxels"])
    assert np.array_equal(O.active_coords(g), golden_grids[f"{name}/active_coords"])
    assert np.array_equal(O.coord_to_index(g, golden_grids[f"{name}/probe"]), golden_grids[f"{name}/probe_index"])
    g2 = O.coarsen(g, 2)
    for f in FIELDS:
        assert np.array_equal(getattr(g2, f), golden_grids[f"{name}/coarse2/{f}"]), f


def test_oracle_points_path(golden_grids):
    p = golden_grids["points/points"]
    vs, og = golden_grids["points/voxel_size"], golden_grids["points/origin"]
    assert np.array_equal(O.quantize(p, vs, og), golden_grids["points/quantized"])
    g = O.build_from_points(p, vs, og)
    for f in FIELDS:
        assert np.array_equal(getattr(g, f), golden_grids[f"points/{f}"]), f


def test_oracle_reference_fixtures(golden_fixtures):
    fx = golden_fixtures
    g = O.build_from_points(fx["points"], fx["voxel_size"], fx["origin"])
    assert list(g.counts) == fx["counts"].tolist()
    assert np.array_equal(O.active_coords(g), fx["active_coords"])
    assert np.array_equal(O.coord_to_index(g, fx["probe_coords"]), fx["probe_expected"])
    ins, outs = O.kernel_map(g, g, 1)
    out = O.conv_igemm(fx["conv_features"], fx["conv_weights"], ins, outs, g.num_voxels)
    # float goldens are BLAS-dependent: tolerance, not bitwise
    assert np.abs(out - fx["conv_expected"]).max() <= 1e-12 * max(1.0, np.abs(fx["conv_expected"]).max())


@pytest.mark.parametrize("name", KMAP_CASES)
@pytest.mark.parametrize("stride", [1, 2])
def test_oracle_kernel_maps_match_reference(golden_grids, golden_kmaps, name, stride):
    g = _grid(golden_grids, name)
    go = g if stride == 1 else O.coarsen(g, 2)
    ins, outs = O.kernel_map(g, go, stride)
    key = f"{name}/s{stride}"
    assert np.array_equal([len(o) for o in outs], golden_kmaps[f"{key}/counts"])
    assert np.array_equal(np.concatenate(ins), golden_kmaps[f"{key}/in_rows"])
    assert np.array_equal(np.concatenate(outs), golden_kmaps[f"{key}/out_rows"])


@pytest.mark.parametrize("name", CONV_CASES)
@pytest.mark.parametrize("stride", [1, 2])
def test_oracle_conv_matches_reference(golden_grids, golden_convs, name, stride):
    g = _grid(golden_grids, name)
    go_grid = g if stride == 1 else O.coarsen(g, 2)
    ins, outs = O.kernel_map(g, go_grid, stride)
    k = f"{name}/s{stride}"
    f, w, go = golden_convs[f"{k}/features"], golden_convs[f"{k}/weights"], golden_convs[f"{k}/grad_out"]
    out = O.conv_igemm(f, w, ins, outs, go_grid.num_voxels)
    ref = golden_convs[f"{k}/out_f64"]
    assert np.abs(out - ref).max() <= 1e-12 * np.abs(ref).max()
    gi, gw = O.conv_backward(ins, outs, go, f, w)
    assert np.abs(gi - golden_convs[f"{k}/grad_in_f64"]).max() <= 1e-12 * np.abs(gi).max()
    assert np.abs(gw - golden_convs[f"{k}/grad_w_f64"]).max() <= 1e-12 * np.abs(gw).max()
    dense = O.conv_dense(g, f, w, go_grid, stride)
    assert np.abs(dense - ref).max() <= 1e-12 * np.abs(ref).max()


def test_oracle_transpose_is_adjoint(golden_grids):
    """<conv_s2(x), y> == <x, conv_transpose(y)>."""
    rng = np.random.default_rng(3)
    g = _grid(golden_grids, "clustered")
    g2 = O.coarsen(g, 2)
    ins, outs = O.kernel_map(g, g2, 2)
    w = rng.normal(size=(7, 5, 3, 3, 3))
    x = rng.normal(size=(g.num_voxels, 5))
    y = rng.normal(size=(g2.num_voxels, 7))
    lhs = np.sum(O.conv_igemm(x, w, ins, outs, g2.num_voxels) * y)
    rhs = np.sum(x * O.conv_transpose(ins, outs, y, w, g.num_voxels))
    assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), 1.0)


def test_oracle_error_messages():
    with pytest.raises(ValueError, match=r"coordinate out of range at row 1: \(0, 1073741825, 0\)"):
        O.build_from_coords([[0, 0, 0], [0, (1 << 30) + 1, 0]])
    with pytest.raises(ValueError, match=r"non-finite point at row 2"):
        O.build_from_points([[0, 0, 0], [1, 1, 1], [np.nan, 0, 0]], [1.0] * 3, [0.0] * 3)
    with pytest.raises(ValueError, match="stride"):
        g = O.build_from_coords([[0, 0, 0]])
        O.kernel_map(g, g, 3)
