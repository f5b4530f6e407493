"""Exact-precision (fp32) gather conv on cfg1 (100K-point cloud, 32->32) and the cfg2 shell (64->64) under
FVDB_EXACT_SKIP = none / masks / sort: median of 20 event-timed launches; results must be bitwise equal."""
import json, os, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2407_01781_b200 as P  # noqa: E402
from paper_2407_01781_b200.conv import gather_conv  # noqa: E402
from paper_2407_01781_b200.workloads import sphere_shell_coords  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


cfg = bench.CONFIGS["cfg1"]
_, points = bench.make_coords(cfg, 0)
g1, _ = P.build_from_points(points, P.VoxelTransform.uniform(0.05))
g2, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
for name, g, C in (("cfg1_32x32", g1, 32), ("cfg2_shell_64x64", g2, 64)):
    km = P.build_kernel_map(g, g, 1)
    x = torch.randn(g.num_voxels, C, device="cuda")
    w = torch.randn(C, C, 3, 3, 3, device="cuda") / (27 * C) ** 0.5
    res, out = {}, {}
    for mode in ("none", "masks", "sort"):
        os.environ["FVDB_EXACT_SKIP"] = mode
        out[mode] = gather_conv(x, km.fwd, w)
        res[mode] = timed(lambda: gather_conv(x, km.fwd, w))
    print(json.dumps({"case": name, "rows": g.num_voxels, "pairs_per_row": round(km.total_pairs / g.num_voxels, 2),
                      "ms": res, "bitwise_equal": all(torch.equal(out["none"], out[m]) for m in out)}), flush=True)
