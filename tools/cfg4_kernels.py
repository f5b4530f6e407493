"""Kernels launched by one cfg4 step (torch.profiler): name, launches per step, device us per step."""
import collections
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2407_01781_b200 as P  # noqa: E402
from paper_2407_01781_b200.workloads import sphere_shell_coords  # noqa: E402

coords = sphere_shell_coords(470, 1.5)
dev = torch.device("cuda")
pts = torch.from_numpy(coords.astype("float64")).to(dev)
tf = P.VoxelTransform.uniform(1.0)
down = P.SparseConv3d(64, 128, stride=2).to(dev)
up = P.SparseConv3d(128, 64, stride=2, transposed=True).to(dev)
x = torch.randn(coords.shape[0], 64, device=dev).to(torch.bfloat16)


def step():
    g, _ = P.build_from_points(pts, tf)
    fine = P.GridBatch([g])
    coarse, h = down(fine, fine.jagged(x))
    _, y = up(coarse, h, out_grid=fine)
    y.jdata.sum(dtype=torch.float32).backward()


for _ in range(5):
    step()
torch.cuda.synchronize()
N = 5
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(N):
        step()
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        a = agg[e.name[:90]]
        a[0] += 1
        a[1] += (e.time_range.end - e.time_range.start)
for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{n / N:5.1f}  {us / N:8.1f} us  {name}")
