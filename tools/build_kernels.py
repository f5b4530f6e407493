"""Per-kernel device time of one build_from_points (cfg4: the cfg2 shell as f64 voxel centres) and one coarsen."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import sphere_shell_coords
pts = torch.from_numpy(sphere_shell_coords(470, 1.5).astype(np.float64)).cuda()
tf = P.VoxelTransform.uniform(1.0)
for _ in range(3):
    g, _ = P.build_from_points(pts, tf)
    P.coarsen(g, 2)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    g, _ = P.build_from_points(pts, tf)
    P.coarsen(g, 2)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
