"""Empty (tile, offset) stages and lane fill of halo plans (cfg2 shell, cfg3 LiDAR, cfg5 shell).

A stage is empty when none of its 128 lanes has a pair; those stages still cost a build, 4-8 MMAs and a
ring slot in k_conv_halo today.  Reads the plan's tile records (u16 local table, kNoSlot = 0xFFFF).
"""
import json, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import lidar_scan_points, sphere_shell_coords


def stats(name, g, K, N):
    km = P.build_kernel_map(g, g, 1)
    for tname, tab in (("fwd", km.fwd),):
        plan = tab.halo_plan(K, N)
        rec = plan.tensors["tile_rec"].view(torch.uint8).reshape(-1, 7424)[:, :6912].contiguous()
        lt = rec.view(torch.int16).reshape(-1, 27, 128)
        has = lt != -1  # 0xFFFF as int16
        per_stage = has.sum(-1)
        empty = (per_stage == 0).float().mean().item()
        fill = (per_stage[per_stage > 0].float() / 128).mean().item()
        print(json.dumps({"cfg": name, "table": tname, "voxels": g.num_voxels, "tiles": int(lt.shape[0]),
                          "empty_stage_frac": round(empty, 4), "lane_fill_nonempty": round(fill, 4),
                          "pairs_per_voxel": round(km.total_pairs / g.num_voxels, 2)}))


g2, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
stats("cfg2", g2, 64, 64)
g3, _ = P.build_from_points(lidar_scan_points(0), P.VoxelTransform.uniform(0.05))
stats("cfg3", g3, 128, 128)
g5, _ = P.build_from_coords(sphere_shell_coords(2048, 1.5))
stats("cfg5", g5, 32, 32)
