"""Per-kernel device time of the cfg1 step (fp32 exact forward, 100K LiDAR points, 32->32)."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402
import bench  # noqa: E402
import paper_2407_01781_b200 as P  # noqa: E402
from paper_2407_01781_b200.conv import gather_conv  # noqa: E402

cfg = bench.CONFIGS["cfg1"]
coords, points = bench.make_coords(cfg, 0)
grid, _ = P.build_from_points(points, P.VoxelTransform.uniform(0.05))
km = P.build_kernel_map(grid, grid, 1)
x = torch.randn(grid.num_voxels, cfg["cin"], device="cuda")
w = torch.randn(cfg["cout"], cfg["cin"], 3, 3, 3, device="cuda") / (27 * cfg["cin"]) ** 0.5
for _ in range(5):
    gather_conv(x, km.fwd, w)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(10):
        gather_conv(x, km.fwd, w)
    torch.cuda.synchronize()
print(grid.num_voxels, km.total_pairs)
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=8))
