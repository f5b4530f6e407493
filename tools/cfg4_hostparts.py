"""Host time of the pieces of the cfg4 step's grid build and coarsen (perf_counter around each call; the device
work is queued, the plan calls include their read-back wait)."""
import collections, json, pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200 import _lib, build as B
from paper_2407_01781_b200.workloads import sphere_shell_coords

acc = collections.defaultdict(float)
L = _lib.lib()


def wrap(name, fn):
    def w(*a, **k):
        t = time.perf_counter()
        r = fn(*a, **k)
        acc[name] += time.perf_counter() - t
        return r
    return w


for n in ("fvdb_build_plan2", "fvdb_build_fill", "fvdb_quantize_points_async", "fvdb_coarsen2_plan",
          "fvdb_coarsen2_fill", "fvdb_build_workspace_bytes", "fvdb_coarsen2_workspace_bytes",
          "fvdb_build_leaf_plan", "fvdb_build_leaf_fill", "fvdb_build_leaf_workspace_bytes"):
    setattr(L, n, wrap(n, getattr(L, n)))
B._alloc_arrays = wrap("_alloc_arrays", B._alloc_arrays)
_lib.workspace = wrap("workspace", _lib.workspace)
pts = torch.from_numpy(sphere_shell_coords(470, 1.5).astype(np.float64)).cuda()
tf = P.VoxelTransform.uniform(1.0)
for _ in range(5):
    g, _ = P.build_from_points(pts, tf)
    P.coarsen(g, 2)
torch.cuda.synchronize()
acc.clear()
N = 50
t0 = time.perf_counter()
for _ in range(N):
    tb = time.perf_counter()
    g, _ = P.build_from_points(pts, tf)
    acc["build_from_points (total)"] += time.perf_counter() - tb
    tc = time.perf_counter()
    P.coarsen(g, 2)
    acc["coarsen (total)"] += time.perf_counter() - tc
torch.cuda.synchronize()
acc["loop"] = time.perf_counter() - t0
print(json.dumps({k: round(v / N * 1e3, 4) for k, v in acc.items()}, indent=1))
