"""N cfg4 U-Net steps (for an ncu launch list: device time per step)."""
import pathlib, sys
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
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    g, _ = P.build_from_points(pts, tf)
    fine = P.GridBatch([g])
    coarse, h = down(fine, fine.jagged(x))
    _, y = up(coarse, h, out_grid=fine)
    y.jdata.sum(dtype=torch.float32).backward()
torch.cuda.synchronize()
