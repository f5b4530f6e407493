"""cfg4 U-Net step: wall vs device time and the host-side hot spots (cProfile over 20 steps)."""
import cProfile, pathlib, pstats, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import sphere_shell_coords
dev = torch.device("cuda")
coords = sphere_shell_coords(470, band=1.5)
pts = torch.from_numpy(coords.astype(np.float64)).to(dev)
tf = P.VoxelTransform.uniform(1.0)
down = P.SparseConv3d(64, 128, stride=2).to(dev)
up = P.SparseConv3d(128, 64, stride=2, transposed=True).to(dev)
x = torch.randn(coords.shape[0], 64, device=dev)

def step():
    g, _ = P.build_from_points(pts, tf)
    fine = P.GridBatch([g])
    coarse, h = down(fine, fine.jagged(x))
    _, y = up(coarse, h, out_grid=fine)
    y.jdata.sum(dtype=torch.float32).backward()

for _ in range(10):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    step()
torch.cuda.synchronize()
print("wall ms/step", (time.perf_counter() - t0) / 20 * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(20):
    step()
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
