"""One cfg2 kernel map (for an ncu capture of k_kernel_map)."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import lidar_scan_points, sphere_shell_coords
which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if which == "cfg3":
    b, _ = P.build_from_points(P.jagged_from_list([torch.from_numpy(lidar_scan_points(s)) for s in range(8)]),
                               P.VoxelTransform.uniform(0.05))
    for _ in range(2):
        P.build_batch_kernel_map(b, b, 1)
else:
    g, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
    for _ in range(2):
        P.build_kernel_map(g, g, 1)
torch.cuda.synchronize()
