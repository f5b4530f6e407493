"""GPU: U-Net glue kernels (csrc/glue.cu) against the reference's golden vectors — bit-exact.

pool 'avg' accumulates in float64 over each coarse voxel's children in ascending fine-row order (the
reference's np.add.at order, conv.py:419-423), so float32 / float64 results are bit-identical; 'max',
subdivide, dilate and upsample_nearest are exact by construction.  Cases mirror the reference's tests
(test_conv.py:271-366, test_build.py:199-215).
"""
import numpy as np
import pytest
import torch

import paper_2407_01781_b200 as P
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gl():
    with np.load(GOLDEN / "glue.npz") as z:
        return {k: z[k] for k in z.files}


def np_(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("factor", [2, 3])
@pytest.mark.parametrize("mode", ["avg", "max"])
def test_pool_bit_exact(gl, factor, mode):
    g, _ = P.build_from_coords(gl["pool/coords"])
    for dt in ("f64", "f32"):
        cg, cf = P.pool(g, gl[f"pool/f{factor}/{dt}"], factor, mode)
        assert np.array_equal(np_(cg.active_coords()), gl[f"pool/f{factor}/{mode}/coarse_coords"])
        want = gl[f"pool/f{factor}/{mode}/{dt}"]
        got = np_(cf)
        assert got.dtype == want.dtype and np.array_equal(got, want), (dt, np.abs(got - want).max())


def test_pool_examples_and_identity():
    g, _ = P.build_from_coords([(0, 0, 0), (4, 4, 4)])
    cg, cf = P.pool(g, np.array([[1.0], [2.0]]), 1)
    assert np.array_equal(np_(cf), [[1.0], [2.0]])
    cube = np.stack(np.meshgrid(*[np.arange(2)] * 3, indexing="ij"), -1).reshape(-1, 3)
    g, _ = P.build_from_coords(cube)
    vals = np.arange(1.0, 9.0).reshape(8, 1)
    assert np_(P.pool(g, vals, 2, mode="max")[1]).tolist() == [[8.0]]
    assert np_(P.pool(g, vals, 2, mode="avg")[1]).tolist() == [[4.5]]
    g, _ = P.build_from_coords([(0, 0, 0), (1, 1, 1)])
    assert np_(P.pool(g, np.array([[3.0], [5.0]]), 2, mode="avg")[1]).tolist() == [[4.0]]
    with pytest.raises(ValueError, match="pool mode"):
        P.pool(g, np.zeros((2, 1)), 2, mode="sum")
    with pytest.raises(ValueError, match="features rows"):
        P.pool(g, np.zeros((3, 1)), 2)


@pytest.mark.parametrize("factor", [2, 3])
def test_subdivide_and_upsample_bit_exact(gl, factor):
    coarse, _ = P.build_from_coords(gl[f"up/f{factor}/coarse_coords_in"])
    fine = P.subdivide(coarse, factor)
    assert np.array_equal(np_(fine.active_coords()), gl[f"up/f{factor}/fine_coords"])
    assert np.allclose(fine.transform.voxel_size, gl[f"up/f{factor}/fine_voxel_size"])
    assert np.allclose(fine.transform.origin, gl[f"up/f{factor}/fine_origin"])
    out = P.upsample_nearest(coarse, gl[f"up/f{factor}/features"], factor, fine)
    assert np.array_equal(np_(out), gl[f"up/f{factor}/out"])
    # pool(upsample(x)) recovers x (reference test_conv.py:316-324)
    cg2, back = P.pool(fine, out, factor, mode="avg")
    assert np.array_equal(np_(cg2.active_coords()), np_(coarse.active_coords()))
    assert np.allclose(np_(back), gl[f"up/f{factor}/features"])
    g, _ = P.build_from_coords(gl["sub/coords"])
    assert np.array_equal(np_(P.subdivide(g, factor).active_coords()), gl[f"sub/f{factor}/active"])
    assert np.array_equal(np_(P.coarsen(P.subdivide(g, factor), factor).active_coords()), gl[f"sub/f{factor}/back"])


@pytest.mark.parametrize("r", [1, 2])
def test_dilate(gl, r):
    g, _ = P.build_from_coords(gl["dil/coords"])
    assert np.array_equal(np_(P.dilate(g, r).active_coords()), gl[f"dil/r{r}/active"])
    with pytest.raises(ValueError, match="radius"):
        P.dilate(g, 0)


def test_upsample_identity_orphan_and_bf16():
    g, _ = P.build_from_coords([(0, 0, 0), (2, 0, 0)])
    f = np.array([[1.0], [2.0]])
    assert np.array_equal(np_(P.upsample_nearest(g, f, 1, g)), f)
    coarse, _ = P.build_from_coords([(0, 0, 0)])
    fine, _ = P.build_from_coords([(0, 0, 0), (5, 5, 5)])
    with pytest.raises(ValueError, match=r"\(5, 5, 5\)"):
        P.upsample_nearest(coarse, np.ones((1, 1)), 2, fine)
    # odd row widths (bf16 x 3 channels = 6 bytes) take the byte path of the gather
    x = torch.arange(6, dtype=torch.float32).reshape(2, 3).to(torch.bfloat16)
    assert torch.equal(P.upsample_nearest(g, x, 1, g).cpu(), x)


def test_pool_batch_equals_per_element(gl):
    grids = [P.build_from_coords(gl[f"pb/coords{i}"])[0] for i in (0, 1)]
    gb = P.grid_batch(grids)
    feats = gb.jagged(torch.from_numpy(gl["pb/features"]).cuda())
    cgb, cf = P.pool_batch(gb, feats, 2, mode="avg")
    assert np.array_equal(np_(cf.jdata), gl["pb/out"])
    assert np.array_equal(np_(cf.joffsets), gl["pb/joffsets"])
    with pytest.raises(TypeError):
        P.pool_batch(grids[0], feats, 2)
