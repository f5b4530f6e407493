"""Golden vectors for sample / sample_with_grad / splat FROM THE REFERENCE (interp.py).

Run in the build container: ``python tests/golden/make_golden_interp.py`` -> ``interp.npz``.
"""
import os
import pathlib
import sys

os.environ.setdefault("OMP_NUM_THREADS", "1")
import numpy as np  # noqa: E402

REF = pathlib.Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
import idxgrid as ig  # noqa: E402
from idxgrid.interp import sample, sample_with_grad, splat  # noqa: E402
from idxgrid.jagged import grid_batch, jagged_from_list  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent


def main():
    a = {}
    rng = np.random.default_rng(31)
    cases = {"scattered": rng.integers(-20, 20, size=(900, 3)),
             "clustered": np.concatenate([rng.integers(-4, 4, size=(400, 3)), rng.integers(10, 16, size=(300, 3))])}
    for name, coords in cases.items():
        tf = ig.VoxelTransform(np.array([0.5, 0.5, 0.5]), np.array([0.2, -0.1, 0.05]))
        g, _ = ig.build_from_coords(coords, tf)
        lo, hi = g.bbox()
        pts = g.transform.index_to_world(rng.uniform(lo - 1, hi + 1, size=(300, 3)))
        f64 = rng.normal(size=(g.num_voxels, 3))
        f32 = rng.normal(size=(g.num_voxels, 2)).astype(np.float32)
        pf = rng.normal(size=(300, 4))
        a[f"{name}/coords"], a[f"{name}/points"] = coords, pts
        a[f"{name}/f64"], a[f"{name}/f32"], a[f"{name}/pf"] = f64, f32, pf
        for mode in ("trilinear", "bezier"):
            v, gr = sample_with_grad(g, f64, pts, mode=mode)
            a[f"{name}/{mode}/sample_f64"], a[f"{name}/{mode}/grad_f64"] = v.jdata, gr.jdata
            a[f"{name}/{mode}/sample_f32"] = sample(g, f32, pts, mode=mode).jdata
            a[f"{name}/{mode}/splat"] = splat(g, pts, pf, mode=mode).jdata
            a[f"{name}/{mode}/splat_f32"] = splat(g, pts, pf.astype(np.float32), mode=mode).jdata
    grids = [ig.build_from_coords(c)[0] for c in cases.values()]
    gb = grid_batch(grids)
    pts = jagged_from_list([rng.uniform(-10, 10, size=(40, 3)), rng.uniform(-5, 15, size=(25, 3))])
    feats = gb.jagged(rng.normal(size=(gb.total_voxels, 2)))
    pfe = pts.with_data(rng.normal(size=(pts.num_rows, 2)))
    a["batch/points"], a["batch/p_off"], a["batch/feats"], a["batch/pf"] = pts.jdata, pts.joffsets, feats.jdata, pfe.jdata
    a["batch/sample"] = sample(gb, feats, pts).jdata
    a["batch/splat"] = splat(gb, pts, pfe).jdata
    np.savez_compressed(OUT / "interp.npz", **a)
    print("wrote interp.npz with", len(a), "arrays")


if __name__ == "__main__":
    main()
