"""Python call sites of torch-level host syncs (.item(), .cpu(), ...) in one cfg4 step, via
torch.cuda.set_sync_debug_mode("warn"). Syncs inside libfvdb_b200 (the build's read-backs) are not seen."""
import collections, pathlib, sys, traceback, warnings
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
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
sites = collections.Counter()


def hook(message, category, filename, lineno, file=None, line=None):
    st = [f"{pathlib.Path(f.filename).name}:{f.lineno}:{f.name}" for f in traceback.extract_stack()
          if "paper_2407" in f.filename]
    sites[" <- ".join(reversed(st[-3:]))] += 1


warnings.simplefilter("always")
warnings.showwarning = hook
torch.cuda.set_sync_debug_mode("warn")
step()
torch.cuda.set_sync_debug_mode(0)
for where, n in sites.most_common():
    print(f"{n:3d}  {where}")
