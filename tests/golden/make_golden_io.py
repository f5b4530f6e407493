"""Reference-written FVDBIDX1 grid files + the reference's error messages on corrupted copies.

Run in the build container: ``python tests/golden/make_golden_io.py`` -> ``tests/golden/io/``.
Imports ``idxgrid`` read-only from /root/reference/pkg/src (never copied into this repo).
"""
import json
import pathlib
import sys

import numpy as np

REF = pathlib.Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
import idxgrid as ig  # noqa: E402
from idxgrid.io import GridFileError, load_grid, save_grid  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent / "io"


def main():
    OUT.mkdir(exist_ok=True)
    rng = np.random.default_rng(21)
    cases = {
        "scattered": (rng.integers(-48, 48, size=(2000, 3)), ig.VoxelTransform.uniform(0.5), "scattered"),
        "multi_tile": (np.concatenate([rng.integers(-9000, 9000, size=(300, 3)),
                                       rng.integers(0, 20, size=(300, 3))]), ig.VoxelTransform.uniform(1.0), ""),
        "named_shell": (None, ig.VoxelTransform(np.array([0.1, 0.2, 0.3]), np.array([1.0, -2.0, 3.5])), "shell é"),
    }
    from idxgrid.workloads import sphere_shell_coords
    meta = {}
    for name, (coords, tf, gname) in cases.items():
        if coords is None:
            coords = sphere_shell_coords(40, band=1.5)
        g, _ = ig.build_from_coords(coords, tf, gname)
        np.save(OUT / f"{name}_coords.npy", g.active_coords())
        save_grid(g, OUT / f"{name}.fvdb")
        meta[name] = {"counts": list(map(int, g.counts)), "name": gname,
                      "voxel_size": g.transform.voxel_size.tolist(), "origin": g.transform.origin.tolist()}
    e = ig.empty_grid(ig.VoxelTransform.uniform(2.0), "empty")
    save_grid(e, OUT / "empty.fvdb")
    meta["empty"] = {"counts": [0, 0, 0, 0], "name": "empty"}
    blob = (OUT / "scattered.fvdb").read_bytes()
    bad = {"bad_magic": b"FVDBIDX2" + blob[8:], "bad_version": blob[:8] + (7).to_bytes(4, "little") + blob[12:],
           "truncated": blob[:-13], "trailing": blob + b"\x00\x01", "header_only": blob[:30]}
    errs = {}
    for k, b in bad.items():
        p = OUT / f"{k}.fvdb"
        p.write_bytes(b)
        try:
            load_grid(p)
            errs[k] = None
        except GridFileError as ex:
            errs[k] = str(ex)
    meta["errors"] = errs
    (OUT / "meta.json").write_text(json.dumps(meta, indent=1, ensure_ascii=False))
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
