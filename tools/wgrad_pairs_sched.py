"""Pair-list wgrad at cfg3 (8 LiDAR grids, 128x128): tile-ordered vs linear schedule.

python tools/wgrad_pairs_sched.py          -> per-schedule ms (CUDA events, 20 runs) + stage statistics
python tools/wgrad_pairs_sched.py once     -> one launch per schedule (for an ncu capture)
"""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_01781_b200 as P  # noqa: E402
from paper_2407_01781_b200.workloads import lidar_scan_points  # noqa: E402

C = sys.modules["paper_2407_01781_b200.conv"]
g, _ = P.build_from_points(P.jagged_from_list([torch.from_numpy(lidar_scan_points(s)) for s in range(8)]),
                           P.VoxelTransform.uniform(0.05))
km = P.build_batch_kernel_map(g, g, 1)
n = g.total_voxels
x = torch.randn(n, 128, device="cuda").to(torch.bfloat16)
gy = torch.randn(n, 128, device="cuda").to(torch.bfloat16)
tab = km.fwd
tab.wgrad_uses = 5
C.os.environ["FVDB_WG_PAIRS"] = "force"
once = len(sys.argv) > 1 and sys.argv[1] == "once"
out = {}
ref = None
for sched in ("tiles", "linear"):
    C._WG_PAIRS_SCHED = sched
    gw = C.wgrad(x, gy, tab)
    torch.cuda.synchronize()
    if once:
        continue
    ref = gw if ref is None else ref
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        C.wgrad(x, gy, tab)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    out[sched] = round(float(np.median(ts)), 4)
    out[sched + "_rel_diff"] = float((gw - ref).abs().max() / ref.abs().max())
if not once:
    tp = tab.pair_tile_pos().cpu().numpy().reshape(27, -1).astype(np.int64)
    cnt = np.diff(tp, axis=1)
    pairs = int(cnt.sum())
    out["pairs"] = pairs
    out["stages_linear"] = int(sum((c.sum() + 127) // 128 * 4 for c in cnt))
    for w in (1, 2, 4, 8):
        t = cnt.shape[1] // w * w
        cw = cnt[:, :t].reshape(27, -1, w).sum(2)
        out[f"stages_win{w}"] = int(((cw + 31) // 32).sum())
    out["pairs_per_tile_offset_mean"] = round(pairs / cnt.size, 1)
print(json.dumps(out))
