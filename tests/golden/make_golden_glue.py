"""Golden vectors for the U-Net glue ops (pool / upsample_nearest / subdivide / dilate) FROM THE REFERENCE.

Run in the build container: ``python tests/golden/make_golden_glue.py`` -> ``glue.npz``.
Imports ``idxgrid`` read-only from /root/reference/pkg/src (never copied into this repo); the GPU box
only reads the fixture.  Cases follow the reference's own tests (test_conv.py:271-366, test_build.py:199-215).
"""
import os
import pathlib
import sys

os.environ.setdefault("OMP_NUM_THREADS", "1")
import numpy as np  # noqa: E402

REF = pathlib.Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
import idxgrid as ig  # noqa: E402
from idxgrid.conv import pool, pool_batch, upsample_nearest  # noqa: E402
from idxgrid.jagged import grid_batch  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent


def main():
    a = {}
    rng = np.random.default_rng(9)
    coords = rng.integers(-16, 16, size=(500, 3))
    g, _ = ig.build_from_coords(coords)
    a["pool/coords"] = coords
    for f in (2, 3):
        f64 = rng.normal(size=(g.num_voxels, 2))
        f32 = rng.normal(size=(g.num_voxels, 5)).astype(np.float32)
        a[f"pool/f{f}/f64"], a[f"pool/f{f}/f32"] = f64, f32
        for mode in ("avg", "max"):
            cg, cf = pool(g, f64, f, mode)
            a[f"pool/f{f}/{mode}/f64"] = cf
            a[f"pool/f{f}/{mode}/f32"] = pool(g, f32, f, mode)[1]
            a[f"pool/f{f}/{mode}/coarse_coords"] = cg.active_coords()
    rng = np.random.default_rng(11)
    cc = rng.integers(-6, 6, size=(80, 3))
    coarse, _ = ig.build_from_coords(cc)
    for f in (2, 3):
        fine = ig.subdivide(coarse, f)
        cf = rng.normal(size=(coarse.num_voxels, 3))
        a[f"up/f{f}/coarse_coords_in"] = cc
        a[f"up/f{f}/features"] = cf
        a[f"up/f{f}/fine_coords"] = fine.active_coords()
        a[f"up/f{f}/out"] = upsample_nearest(coarse, cf, f, fine)
        a[f"up/f{f}/fine_voxel_size"] = fine.transform.voxel_size
        a[f"up/f{f}/fine_origin"] = fine.transform.origin
    rng = np.random.default_rng(7)
    sc = rng.integers(-40, 40, size=(400, 3))
    g, _ = ig.build_from_coords(sc)
    a["sub/coords"] = sc
    for f in (2, 3):
        a[f"sub/f{f}/active"] = ig.subdivide(g, f).active_coords()
        a[f"sub/f{f}/back"] = ig.coarsen(ig.subdivide(g, f), f).active_coords()
    small = rng.integers(-5, 5, size=(30, 3))
    gs, _ = ig.build_from_coords(small)
    a["dil/coords"] = small
    for r in (1, 2):
        a[f"dil/r{r}/active"] = ig.dilate(gs, r).active_coords()
    rng = np.random.default_rng(12)
    grids = [ig.build_from_coords(rng.integers(-s, s, size=(n, 3)))[0] for s, n in ((8, 120), (14, 300))]
    gb = grid_batch(grids)
    feats = gb.jagged(rng.normal(size=(gb.total_voxels, 4)))
    a["pb/coords0"], a["pb/coords1"] = grids[0].active_coords(), grids[1].active_coords()
    a["pb/features"] = feats.jdata
    cgb, cfe = pool_batch(gb, feats, 2, mode="avg")
    a["pb/out"] = cfe.jdata
    a["pb/joffsets"] = cfe.joffsets
    np.savez_compressed(OUT / "glue.npz", **a)
    print("wrote glue.npz with", len(a), "arrays")


if __name__ == "__main__":
    main()
