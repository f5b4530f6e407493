"""Halo-plan cost in a loop that rebuilds its map every step (steady state: the caching allocator warm).
Prints per-phase wall / event ms of: kernel map, transposed table, halo plan fwd, halo plan dgrad."""
import json, pathlib, sys, time, cProfile, pstats
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import sphere_shell_coords
c = torch.from_numpy(sphere_shell_coords(470, 1.5)).cuda()
g, _ = P.build_from_coords(c)

def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(); r = fn(); e1.record(); torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) * 1e3, e0.elapsed_time(e1)

res = []
for it in range(8):
    km, w0, d0 = timed(lambda: P.build_kernel_map(g, g, 1))
    bwd, w1, d1 = timed(lambda: km.bwd)
    _, w2, d2 = timed(lambda: km.fwd.halo_plan(64, 64))
    _, w3, d3 = timed(lambda: km.bwd.halo_plan(64, 64))
    res.append({"kmap": (round(w0, 3), round(d0, 3)), "transpose": (round(w1, 3), round(d1, 3)),
                "plan_fwd": (round(w2, 3), round(d2, 3)), "plan_dgrad": (round(w3, 3), round(d3, 3))})
for r in res[-3:]:
    print(json.dumps(r))
pr = cProfile.Profile(); pr.enable()
for _ in range(5):
    km = P.build_kernel_map(g, g, 1); km.fwd.halo_plan(64, 64); km.bwd.halo_plan(64, 64)
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(15)
