"""cProfile of the cfg4 step (host side): top functions by own time and by cumulative time, per step."""
import cProfile
import pathlib
import pstats
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

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


for _ in range(10):
    step()
torch.cuda.synchronize()
N = 50
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    step()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumulative").print_stats(45)
