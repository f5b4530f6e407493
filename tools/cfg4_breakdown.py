"""Phase breakdown of the cfg4 step (U-Net stage incl. grid build): host wall vs device events."""
import json, pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import sphere_shell_coords
from paper_2407_01781_b200.nn import coarsen_batch
from paper_2407_01781_b200.conv import batch_grid_kernel_map

coords = sphere_shell_coords(470, 1.5)
pts = torch.from_numpy(coords.astype(np.float64)).cuda()
tf = P.VoxelTransform.uniform(1.0)
down = P.SparseConv3d(64, 128, stride=2).cuda()
up = P.SparseConv3d(128, 64, stride=2, transposed=True).cuda()
x = torch.randn(coords.shape[0], 64, device="cuda")


def step(mark):
    g, _ = P.build_from_points(pts, tf); mark("build")
    fine = P.GridBatch([g])
    cg = coarsen_batch(fine, 2); mark("coarsen")
    km = batch_grid_kernel_map(fine, cg, 2); mark("kmap_s2")
    _ = km.bwd; mark("transpose")
    coarse, h = down(fine, fine.jagged(x)); mark("down_fwd")
    _, y = up(coarse, h, out_grid=fine); mark("up_fwd")
    y.jdata.sum(dtype=torch.float32).backward(); mark("backward")


for _ in range(3):
    step(lambda n: None)
torch.cuda.synchronize()
res = {}
for rep in range(5):
    evs, walls = [], []
    def mark(name):
        e = torch.cuda.Event(enable_timing=True); e.record(); evs.append((name, e)); walls.append((name, time.perf_counter()))
    mark("start")
    step(mark)
    torch.cuda.synchronize()
    for i in range(1, len(evs)):
        n = evs[i][0]
        res.setdefault(n, []).append((evs[i - 1][1].elapsed_time(evs[i][1]), (walls[i][1] - walls[i - 1][1]) * 1e3))
print(json.dumps({k: {"device_ms": round(float(np.median([a for a, b in v])), 3),
                      "host_ms": round(float(np.median([b for a, b in v])), 3)} for k, v in res.items()}, indent=1))
