"""Time build_kernel_map (neighbour leaves + kernel map + pair counts) on cfg2 (stride 1) and cfg4 (stride 2)."""
import json, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import sphere_shell_coords
g, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
gc = P.coarsen(g, 2)
for name, (gi, go, s) in {"cfg2_s1": (g, g, 1), "cfg4_s2": (g, gc, 2)}.items():
    for _ in range(3):
        P.build_kernel_map(gi, go, s)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); km = P.build_kernel_map(gi, go, s); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[5]
    print(json.dumps({"map": name, "ms": ms, "table_GB_per_s": 27 * go.num_voxels * 4 / ms / 1e6,
                      "pairs": km.total_pairs}))
