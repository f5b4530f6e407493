"""Per-kernel device time of one cfg4 step (torch.profiler / CUPTI), to attribute the step's phases."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import sphere_shell_coords
from paper_2407_01781_b200.nn import coarsen_batch

coords = sphere_shell_coords(470, 1.5)
pts = torch.from_numpy(coords.astype(np.float64)).cuda()
tf = P.VoxelTransform.uniform(1.0)
down = P.SparseConv3d(64, 128, stride=2).cuda()
up = P.SparseConv3d(128, 64, stride=2, transposed=True).cuda()
x = torch.randn(coords.shape[0], 64, device="cuda")


def step():
    g, _ = P.build_from_points(pts, tf)
    fine = P.GridBatch([g])
    coarse, h = down(fine, fine.jagged(x))
    _, y = up(coarse, h, out_grid=fine)
    y.jdata.float().sum().backward()


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
