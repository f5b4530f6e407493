"""Generate golden vectors for the hot path FROM THE REFERENCE ITSELF.

Run in the build container (where the read-only reference checkout exists):

    python tests/golden/make_golden.py

It imports ``idxgrid`` from /root/reference/pkg/src (never copied into this repo),
runs the reference on seeded inputs and writes small ``.npz`` fixtures next to
this script.  The fixtures travel with the repo; nothing at test / bench time on
the GPU box reads /root/reference.

Fixture files:
  fixtures_ref.npz  — the reference's own frontend/test/fixtures.json, decoded
                      (build counts, active coords, coord→index probes, igemm conv f64)
  grids.npz         — full topology arrays of seeded grids (bit-exact targets)
  kmaps.npz         — per-offset kernel maps, stride 1 and stride 2
  convs.npz         — conv forward / backward outputs (f64 and f32) incl. stride 2
  sizes.json        — voxel / leaf / pair counts of the full-size bench configs
"""

from __future__ import annotations

import base64
import json
import os
import pathlib
import sys

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np

REF = pathlib.Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2]))

import idxgrid as ig  # noqa: E402  (reference, read-only)
from idxgrid.conv import build_kernel_map, conv, conv_backward  # noqa: E402
from idxgrid.workloads import random_points, sphere_shell_coords  # noqa: E402

from paper_2407_01781_b200.workloads import lidar_scan_points  # noqa: E402  (input generator)

OUT = pathlib.Path(__file__).resolve().parent
FIELDS = ("tile_keys", "upper_origins", "upper_child_starts", "lower_offset_in_upper",
          "lower_origins", "lower_child_starts", "leaf_offset_in_lower", "leaf_keys",
          "leaf_origins", "leaf_masks", "leaf_prefix", "leaf_value_offset")


def unwire(w):
    raw = base64.b64decode(w["data"])
    return np.frombuffer(raw, dtype=np.dtype(w["dtype"]).newbyteorder("<")).reshape(w["shape"]).copy()


def grid_cases():
    """Seeded coordinate sets covering the reference's build edge cases."""
    rng = np.random.default_rng(1234)
    cases = {
        "scattered": rng.integers(-48, 48, size=(2000, 3)),
        "dup_heavy": rng.integers(-3, 3, size=(500, 3)),
        "single": np.array([[5, -7, 9]]),
        "pair": np.array([[0, 0, 0], [1, 0, 0]]),
        "multi_tile": rng.integers(-9000, 9000, size=(3000, 3)),
        "wide": rng.integers(-(1 << 30), (1 << 30) + 1, size=(1000, 3)),
        "neg_boundary": np.array([[-1, -1, -1], [0, 0, 0], [-4096, 4095, -4097],
                                  [-(1 << 30), (1 << 30), 0], [7, 8, -8], [-8, -9, 127],
                                  [128, -129, 4096]]),
        "shell": ig.workloads.sphere_shell_coords(64, band=1.5),
        "small_shell": ig.workloads.sphere_shell_coords(28, band=1.5),
        "clustered": np.concatenate([c + np.round(rng.normal(0, 3.0, (60, 3))).astype(np.int64)
                                     for c in rng.integers(-40, 40, size=(6, 3))]),
    }
    return cases


def main():
    # 1. the reference's shared fixtures (frontend/test/make_fixtures.py:28-71)
    fx = json.loads((REF / "frontend/test/fixtures.json").read_text())
    np.savez_compressed(
        OUT / "fixtures_ref.npz",
        points=unwire(fx["build"]["points"]),
        voxel_size=np.array(fx["build"]["voxel_size"], np.float64),
        origin=np.array(fx["build"]["origin"], np.float64),
        counts=np.array(fx["build"]["counts"], np.int64),
        probe_coords=unwire(fx["coord_to_index"]["coords"]),
        probe_expected=unwire(fx["coord_to_index"]["expected"]),
        active_coords=unwire(fx["active_coords"]["expected"]),
        conv_features=unwire(fx["sample"]["features"]),
        conv_weights=unwire(fx["conv"]["weights"]),
        conv_expected=unwire(fx["conv"]["expected"]),
    )

    # 2. grids: full topology arrays
    g_arrays = {}
    for name, c in grid_cases().items():
        g, _ = ig.build_from_coords(c)
        g_arrays[f"{name}/coords"] = np.asarray(c, np.int64)
        for f in FIELDS:
            g_arrays[f"{name}/{f}"] = getattr(g, f)
        g_arrays[f"{name}/num_voxels"] = np.array(g.num_voxels)
        g_arrays[f"{name}/active_coords"] = g.active_coords()
        g2 = ig.coarsen(g, 2)
        for f in FIELDS:
            g_arrays[f"{name}/coarse2/{f}"] = getattr(g2, f)
        g_arrays[f"{name}/coarse2/num_voxels"] = np.array(g2.num_voxels)
        probe = np.concatenate([np.asarray(c, np.int64)[:300],
                                np.random.default_rng(7).integers(-60, 60, size=(300, 3))])
        g_arrays[f"{name}/probe"] = probe
        g_arrays[f"{name}/probe_index"] = g.coord_to_index_many(probe)
    # points path (quantize + build), incl. the exact .5 rounding case (test_build.py:107-112)
    rng = np.random.default_rng(99)
    pts = np.concatenate([random_points(rng, 3000, sigma=1.0),
                          np.array([[0.5, -0.5, 1.5], [2.4999999999999996, -2.5, 0.25]])])
    t = ig.VoxelTransform(np.array([0.05, 0.07, 0.1]), np.array([0.01, -0.02, 0.3]))
    g, _ = ig.build_from_points(pts, t)
    g_arrays["points/points"] = pts
    g_arrays["points/voxel_size"] = t.voxel_size
    g_arrays["points/origin"] = t.origin
    g_arrays["points/quantized"] = t.quantize(pts)
    for f in FIELDS:
        g_arrays[f"points/{f}"] = getattr(g, f)
    g_arrays["points/num_voxels"] = np.array(g.num_voxels)
    np.savez_compressed(OUT / "grids.npz", **g_arrays)

    # 3. kernel maps
    k_arrays = {}
    cases = grid_cases()
    for name in ("scattered", "shell", "clustered", "multi_tile", "neg_boundary", "pair"):
        g, _ = ig.build_from_coords(cases[name])
        for stride in (1, 2):
            go = g if stride == 1 else ig.coarsen(g, 2)
            km = build_kernel_map(g, go, stride)
            k_arrays[f"{name}/s{stride}/counts"] = km.pair_counts
            k_arrays[f"{name}/s{stride}/in_rows"] = np.concatenate(km.in_rows)
            k_arrays[f"{name}/s{stride}/out_rows"] = np.concatenate(km.out_rows)
    np.savez_compressed(OUT / "kmaps.npz", **k_arrays)

    # 4. conv forward/backward outputs
    c_arrays = {}
    rng = np.random.default_rng(5)
    for name, cin, cout in (("scattered", 8, 16), ("small_shell", 16, 24), ("clustered", 5, 7)):
        g, _ = ig.build_from_coords(cases[name])
        for stride in (1, 2):
            go_grid = g if stride == 1 else ig.coarsen(g, 2)
            km = build_kernel_map(g, go_grid, stride)
            f64 = rng.normal(size=(g.num_voxels, cin))
            w64 = rng.normal(size=(cout, cin, 3, 3, 3)) / np.sqrt(27 * cin)
            go64 = rng.normal(size=(go_grid.num_voxels, cout))
            key = f"{name}/s{stride}"
            c_arrays[f"{key}/features"] = f64
            c_arrays[f"{key}/weights"] = w64
            c_arrays[f"{key}/grad_out"] = go64
            c_arrays[f"{key}/out_f64"] = conv(g, f64, w64, grid_out=go_grid, stride=stride, kmap=km)
            gi, gw = conv_backward(km, go64, f64, w64)
            c_arrays[f"{key}/grad_in_f64"] = gi
            c_arrays[f"{key}/grad_w_f64"] = gw
            f32, w32, go32 = (a.astype(np.float32) for a in (f64, w64, go64))
            c_arrays[f"{key}/out_f32"] = conv(g, f32, w32, grid_out=go_grid, stride=stride, kmap=km)
            gi, gw = conv_backward(km, go32, f32, w32)
            c_arrays[f"{key}/grad_in_f32"] = gi
            c_arrays[f"{key}/grad_w_f32"] = gw
    np.savez_compressed(OUT / "convs.npz", **c_arrays)

    # 5. full-size config statistics (bit-exact counts the GPU must reproduce)
    sizes = {}
    pts = random_points(np.random.default_rng(0), 100_000, sigma=1.0)
    g, _ = ig.build_from_points(pts, ig.VoxelTransform.uniform(0.05))
    km = build_kernel_map(g, g, 1)
    sizes["cfg1"] = {"counts": list(g.counts), "pairs": km.total_pairs,
                     "pair_counts": km.pair_counts.tolist()}
    c = sphere_shell_coords(470, band=1.5)
    g, _ = ig.build_from_coords(c)
    km = build_kernel_map(g, g, 1)
    ac = g.active_coords()
    sizes["cfg2"] = {"counts": list(g.counts), "pairs": km.total_pairs,
                     "pair_counts": km.pair_counts.tolist(),
                     "coord_checksum": int((ac * np.array([1, 7919, 104729])).sum() % (1 << 61)),
                     "leaf_mask_xor": int(np.bitwise_xor.reduce(g.leaf_masks.ravel()))}
    g2 = ig.coarsen(g, 2)
    km2 = build_kernel_map(g, g2, 2)
    sizes["cfg4"] = {"fine_counts": list(g.counts), "coarse_counts": list(g2.counts),
                     "pairs_s2": km2.total_pairs, "pair_counts_s2": km2.pair_counts.tolist()}
    lid = []
    for seed in (0, 1):
        g, _ = ig.build_from_points(lidar_scan_points(seed), ig.VoxelTransform.uniform(0.05))
        km = build_kernel_map(g, g, 1)
        lid.append({"seed": seed, "counts": list(g.counts), "pairs": km.total_pairs})
    sizes["cfg3"] = lid
    (OUT / "sizes.json").write_text(json.dumps(sizes, indent=1))
    print("wrote", sorted(p.name for p in OUT.glob("*.npz")), "and sizes.json")


if __name__ == "__main__":
    main()
