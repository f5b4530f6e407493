"""Full-size golden digests of every BASELINE config, FROM THE REFERENCE ITSELF (VERDICT r1 "next" #1).

Run in the build container (read-only reference checkout at /root/reference):

    python tests/golden/make_golden_fullsize.py [cfg1 cfg2 cfg3 cfg4 cfg5]

Inputs come from the repo's deterministic generators (the same calls bench.py makes); the reference builds
the grids (build.py:82-230, coarsen :325-339) and the kernel maps (conv.py:105-122).  Written to
``fullsize.json``: per grid the SHA-256 of each of the 12 topology arrays and of active_coords() (voxel
order), per map the SHA-256 of its per-offset (in_rows, out_rows) lists (tests/fullsize_hash.py).  cfg5
(19.4M voxels, 404M pairs) takes ~4 minutes.
"""
from __future__ import annotations

import json
import os
import pathlib
import sys
import time

os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))

import numpy as np

REF = pathlib.Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import idxgrid as ig  # noqa: E402  (reference, read-only)
from idxgrid.conv import build_kernel_map  # noqa: E402

from fullsize_hash import FIELDS, grid_digest, map_digest  # noqa: E402
from paper_2407_01781_b200.workloads import lidar_scan_points, random_points, sphere_shell_coords  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent / "fullsize.json"


def gd(g):
    return grid_digest({f: getattr(g, f) for f in FIELDS}, g.active_coords(), g.counts)


def md(km):
    return map_digest(km.in_rows, km.out_rows, km.pair_counts)


def main(which):
    res = json.loads(OUT.read_text()) if OUT.exists() else {}
    t0 = time.time()
    if "cfg1" in which:
        pts = random_points(np.random.default_rng(0), 100_000, sigma=1.0)
        g, _ = ig.build_from_points(pts, ig.VoxelTransform.uniform(0.05))
        res["cfg1"] = {"grid": gd(g), "map": md(build_kernel_map(g, g, 1))}
        print("cfg1", time.time() - t0, flush=True)
    if "cfg2" in which:
        g, _ = ig.build_from_coords(sphere_shell_coords(470, band=1.5))
        res["cfg2"] = {"grid": gd(g), "map": md(build_kernel_map(g, g, 1))}
        print("cfg2", time.time() - t0, flush=True)
    if "cfg3" in which:
        res["cfg3"] = []
        for seed in range(8):
            g, _ = ig.build_from_points(lidar_scan_points(seed), ig.VoxelTransform.uniform(0.05))
            res["cfg3"].append({"seed": seed, "grid": gd(g), "map": md(build_kernel_map(g, g, 1))})
        print("cfg3", time.time() - t0, flush=True)
    if "cfg4" in which:
        pts = sphere_shell_coords(470, band=1.5).astype(np.float64)
        g, _ = ig.build_from_points(pts, ig.VoxelTransform.uniform(1.0))
        c = ig.coarsen(g, 2)
        res["cfg4"] = {"fine": gd(g), "coarse": gd(c), "map_s2": md(build_kernel_map(g, c, 2)),
                       "map_coarse_s1": md(build_kernel_map(c, c, 1))}
        print("cfg4", time.time() - t0, flush=True)
    if "cfg5" in which:
        g, _ = ig.build_from_coords(sphere_shell_coords(2048, band=1.5))
        print("cfg5 grid", time.time() - t0, flush=True)
        res["cfg5"] = {"grid": gd(g)}
        OUT.write_text(json.dumps(res, indent=1))
        res["cfg5"]["map"] = md(build_kernel_map(g, g, 1))
        print("cfg5", time.time() - t0, flush=True)
    OUT.write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
