"""Kernel-map stage on cfg2 (stride 1), cfg4 (stride 2) and the cfg3 batch: events around build_kernel_map
(host launch overhead included) and a cProfile of the host side (where the non-device time goes).
Run under ncu for the per-kernel device times."""
import cProfile, json, pathlib, pstats, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import lidar_scan_points, sphere_shell_coords
g, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
gc = P.coarsen(g, 2)
batch, _ = P.build_from_points(P.jagged_from_list([torch.from_numpy(lidar_scan_points(s)) for s in range(8)]),
                               P.VoxelTransform.uniform(0.05))
cases = {"cfg2_s1": lambda: P.build_kernel_map(g, g, 1), "cfg4_s2": lambda: P.build_kernel_map(g, gc, 2),
         "cfg3_batch": lambda: P.build_batch_kernel_map(batch, batch, 1)}
for name, fn in cases.items():
    for _ in range(3):
        fn()
    ts, ws = [], []
    for _ in range(10):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(); km = fn(); b.record(); torch.cuda.synchronize()
        ws.append((time.perf_counter() - t0) * 1e3)
        ts.append(a.elapsed_time(b))
    print(json.dumps({"map": name, "event_ms": sorted(ts)[5], "wall_ms": sorted(ws)[5], "pairs": km.total_pairs}))
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    P.build_kernel_map(g, g, 1)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
