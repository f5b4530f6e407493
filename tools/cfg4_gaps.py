"""Device idle gaps inside the cfg4 step (torch.profiler trace): kernel busy time per step, and the largest gaps
with the kernels on either side (where the host held the device up)."""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2407_01781_b200 as P  # noqa: E402
from paper_2407_01781_b200.workloads import sphere_shell_coords  # noqa: E402

coords = sphere_shell_coords(470, 1.5)
dev = torch.device("cuda")
pts = torch.from_numpy(coords.astype("float64")).to(dev)
tf = P.VoxelTransform.uniform(1.0)
down = P.SparseConv3d(64, 128, stride=2).to(dev)
up = P.SparseConv3d(128, 64, stride=2, transposed=True).to(dev)
x = torch.randn(coords.shape[0], 64, device=dev).to(torch.bfloat16)


def step():
    g, _ = P.build_from_points(pts, tf)
    fine = P.GridBatch([g])
    coarse, h = down(fine, fine.jagged(x))
    _, y = up(coarse, h, out_grid=fine)
    y.jdata.sum(dtype=torch.float32).backward()


for _ in range(5):
    step()
torch.cuda.synchronize()
N = 5
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(N):
        step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
busy = sum(e.time_range.end - e.time_range.start for e in ev) / N
span = (ev[-1].time_range.end - ev[0].time_range.start) / N
gaps = []
for a, b in zip(ev, ev[1:]):
    g = b.time_range.start - a.time_range.end
    if g > 0:
        gaps.append((g, a.name[:50], b.name[:50]))
agg = {}
for g, a, b in gaps:
    k = (a, b)
    agg[k] = agg.get(k, 0) + g / N
top = sorted(agg.items(), key=lambda kv: -kv[1])[:15]
print(json.dumps({"kernels_per_step": len(ev) / N, "busy_us_per_step": round(busy, 1),
                  "span_us_per_step": round(span, 1),
                  "gaps_us_per_step": [[round(v, 1), a, b] for (a, b), v in top]}, indent=1))
