"""Python call sites of every blocking host<->device sync in one cfg4 step (torch.profiler with stacks)."""
import collections, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import sphere_shell_coords

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
    y.jdata.sum(dtype=torch.float32).backward()


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], with_stack=True) as prof:
    step()
    torch.cuda.synchronize()
sites = collections.Counter()
for ev in prof.events():
    if ev.name in ("cudaStreamSynchronize", "cudaDeviceSynchronize", "cudaMemcpyAsync", "cudaMemcpy"):
        st = [f for f in (ev.stack or []) if "paper_2407" in f or "tools/" in f]
        sites[(ev.name, " <- ".join(s.split("/")[-1] for s in st[:3]))] += 1
for (name, where), n in sites.most_common():
    print(f"{n:3d}  {name:24s} {where}")
