"""One bench-like step (fwd, wgrad, dgrad on reused tables: the steady kernels) for an ncu capture.
python tools/ncu_step.py cfg2|cfg3|cfg5"""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.conv import gather_conv, wgrad
from paper_2407_01781_b200.workloads import lidar_scan_points, sphere_shell_coords
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if cfg == "cfg3":
    g, _ = P.build_from_points(P.jagged_from_list([torch.from_numpy(lidar_scan_points(s)) for s in range(8)]),
                               P.VoxelTransform.uniform(0.05))
    km = P.build_batch_kernel_map(g, g, 1)
    n, C = g.total_voxels, 128
else:
    g, _ = P.build_from_coords(sphere_shell_coords(2048 if cfg == "cfg5" else 470, 1.5))
    km = P.build_kernel_map(g, g, 1)
    n, C = g.num_voxels, 32 if cfg == "cfg5" else 64
x = torch.randn(n, C, device="cuda").to(torch.bfloat16)
gy = torch.randn(n, C, device="cuda").to(torch.bfloat16)
w = torch.randn(C, C, 3, 3, 3, device="cuda") / (27 * C) ** 0.5
for _ in range(6):
    gather_conv(x, km.fwd, w)
    wgrad(x, gy, km.fwd)
    gather_conv(gy, km.bwd, w, transpose=True)
torch.cuda.synchronize()
