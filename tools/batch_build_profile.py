"""cfg3 batched build (8 LiDAR grids, 2.1M points): wall / event time and host hot spots."""
import cProfile, pathlib, pstats, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import lidar_scan_points
jag = P.jagged_from_list([torch.from_numpy(lidar_scan_points(s)).cuda() for s in range(8)])
tf = P.VoxelTransform.uniform(0.05)
for _ in range(3):
    b, _ = P.build_from_points(jag, tf)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    b = None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b, _ = P.build_from_points(jag, tf)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
print("batched build wall ms", sorted(ts))
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s in range(8):
        P.build_from_points(jag.element(s), tf)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
print("8 single builds wall ms", sorted(ts))
pr = cProfile.Profile(); pr.enable()
for _ in range(5):
    b, _ = P.build_from_points(jag, tf)
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
