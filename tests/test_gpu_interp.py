"""GPU: sample / sample_with_grad / splat (csrc/interp.cu) against golden vectors produced by the reference
(tests/golden/make_golden_interp.py; reference interp.py:44-203) plus the reference's own property tests
(test_interp.py): voxel-centre and midpoint values, out-of-grid zeros, partition of unity, adjoint identity,
determinism, batch == per element, dtype preservation, error texts.

Tolerances: f64 sample / gradient / splat rel <= 1e-12 (same weights and f64 accumulation; the reference's
einsum / reduceat may sum in a different association); f32 outputs within one f32 ulp-scale rel 1e-6.
"""
import numpy as np
import pytest
import torch

import paper_2407_01781_b200 as P
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gi():
    with np.load(GOLDEN / "interp.npz") as z:
        return {k: z[k] for k in z.files}


def rel(a, b):
    a = a.detach().double().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.mark.parametrize("name", ["scattered", "clustered"])
@pytest.mark.parametrize("mode", ["trilinear", "bezier"])
def test_matches_reference(gi, name, mode):
    tf = P.VoxelTransform(np.array([0.5, 0.5, 0.5]), np.array([0.2, -0.1, 0.05]))
    g, _ = P.build_from_coords(gi[f"{name}/coords"], tf)
    pts = gi[f"{name}/points"]
    v, gr = P.sample_with_grad(g, gi[f"{name}/f64"], pts, mode=mode)
    assert v.jdata.dtype == torch.float64
    assert rel(v.jdata, gi[f"{name}/{mode}/sample_f64"]) <= 1e-12
    assert rel(gr.jdata, gi[f"{name}/{mode}/grad_f64"]) <= 1e-12
    v32 = P.sample(g, gi[f"{name}/f32"], pts, mode=mode).jdata
    assert v32.dtype == torch.float32 and rel(v32, gi[f"{name}/{mode}/sample_f32"]) <= 1e-6
    sp = P.splat(g, pts, gi[f"{name}/pf"], mode=mode).jdata
    assert rel(sp, gi[f"{name}/{mode}/splat"]) <= 1e-12
    sp32 = P.splat(g, pts, gi[f"{name}/pf"].astype(np.float32), mode=mode).jdata
    assert rel(sp32, gi[f"{name}/{mode}/splat_f32"]) <= 1e-6
    assert torch.equal(sp, P.splat(g, pts, gi[f"{name}/pf"], mode=mode).jdata)  # bitwise reproducible


def test_reference_examples():
    g, _ = P.build_from_coords([(0, 0, 0), (1, 0, 0), (0, 2, 0)])
    f = np.random.default_rng(0).normal(size=(3, 3))
    centers = g.transform.index_to_world(g.active_coords().cpu().numpy())
    assert np.allclose(P.sample(g, f, centers).jdata.cpu().numpy(), f)
    g, _ = P.build_from_coords([(0, 0, 0), (1, 0, 0)])
    assert np.allclose(P.sample(g, np.array([[2.0], [6.0]]), np.array([[0.5, 0.0, 0.0]])).jdata.cpu(), [[4.0]])
    assert np.allclose(P.splat(g, np.array([[0.0, 0.0, 0.0]]), np.array([[5.0, -1.0]])).jdata.cpu(),
                       [[5.0, -1.0], [0.0, 0.0]])
    assert np.allclose(P.splat(g, np.array([[0.5, 0.0, 0.0]]), np.array([[4.0]])).jdata.cpu(), [[2.0], [2.0]])
    g1, _ = P.build_from_coords([(0, 0, 0)])
    assert np.allclose(P.splat(g1, np.array([[0.5, 0.0, 0.0]]), np.array([[4.0]])).jdata.cpu(), [[2.0]])
    assert np.array_equal(P.sample(g1, np.ones((1, 2)), np.array([[50.0, 50.0, 50.0]])).jdata.cpu(), np.zeros((1, 2)))
    assert P.sample(g1, np.ones((1, 1), np.float32), np.zeros((1, 3))).jdata.dtype == torch.float32
    with pytest.raises(ValueError, match="2"):
        P.sample(g, np.ones((5, 1)), np.zeros((1, 3)))
    with pytest.raises(ValueError, match="interpolation mode"):
        P.sample(g, np.ones((2, 1)), np.zeros((1, 3)), mode="cubic")
    with pytest.raises(ValueError, match=r"points must be \[-1,3\]"):
        P.sample(g, np.ones((2, 1)), np.zeros((1, 2)))


@pytest.mark.parametrize("mode", ["trilinear", "bezier"])
def test_unity_adjoint_constant_gradient(mode):
    r = np.arange(-4, 4)
    dense = np.stack(np.meshgrid(r, r, r, indexing="ij"), -1).reshape(-1, 3)
    g, _ = P.build_from_coords(dense)
    rng = np.random.default_rng(4)
    pts = g.transform.index_to_world(rng.uniform(-1, 2, size=(200, 3)))
    ones = P.sample(g, np.ones((g.num_voxels, 1)), pts, mode=mode).jdata.cpu().numpy()
    assert np.abs(ones - 1.0).max() < 1e-12
    _, grads = P.sample_with_grad(g, np.full((g.num_voxels, 2), 3.25), pts, mode=mode)
    assert np.abs(grads.jdata.cpu().numpy()).max() < 1e-12
    pts = g.transform.index_to_world(rng.uniform(-6, 6, size=(60, 3)))
    f = rng.normal(size=(60, 4))
    gg = rng.normal(size=(g.num_voxels, 4))
    lhs = float((P.splat(g, pts, f, mode=mode).jdata.cpu().numpy() * gg).sum())
    rhs = float((f * P.sample(g, gg, pts, mode=mode).jdata.cpu().numpy()).sum())
    assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), abs(rhs), 1e-30)


def test_batch_matches_reference(gi):
    grids = [P.build_from_coords(gi[f"{n}/coords"])[0] for n in ("scattered", "clustered")]
    gb = P.grid_batch(grids)
    off = gi["batch/p_off"]
    pts = P.JaggedTensor(gi["batch/points"], off, np.repeat(np.arange(2), off[:, 1] - off[:, 0]))
    feats = gb.jagged(torch.from_numpy(gi["batch/feats"]).cuda())
    assert rel(P.sample(gb, feats, pts).jdata, gi["batch/sample"]) <= 1e-12
    pf = pts.with_data(gi["batch/pf"])
    assert rel(P.splat(gb, pts, pf).jdata, gi["batch/splat"]) <= 1e-12
    with pytest.raises(ValueError, match="row-aligned"):
        P.splat(gb, pts, P.JaggedTensor(gi["batch/pf"], off[::-1] * 0 + [[0, 25], [25, 65]],
                                        np.repeat(np.arange(2), [25, 40])))
