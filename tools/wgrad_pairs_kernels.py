"""Per-kernel device time (torch.profiler) of one wgrad on the cfg3 LiDAR map, 128->128, table kernel
(FVDB_WG_PAIRS=0) vs pair-list kernel (force). python tools/wgrad_pairs_kernels.py"""
import json, os, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import paper_2407_01781_b200 as P  # noqa: E402
from paper_2407_01781_b200.conv import wgrad  # noqa: E402
from paper_2407_01781_b200.workloads import lidar_scan_points  # noqa: E402

g3, _ = P.build_from_points(lidar_scan_points(0), P.VoxelTransform.uniform(0.05))
tab = P.build_kernel_map(g3, g3, 1).fwd
x = torch.randn(g3.num_voxels, 128, device="cuda").to(torch.bfloat16)
go = torch.randn(tab.n, 128, device="cuda").to(torch.bfloat16)
for mode in ("0", "force"):
    os.environ["FVDB_WG_PAIRS"] = mode
    for _ in range(3):
        wgrad(x, go, tab)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            wgrad(x, go, tab)
        torch.cuda.synchronize()
    ks = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            k = e.name.split("<")[0].split("(")[0][-40:]
            ks[k] = ks.get(k, 0.0) + e.device_time / 5
    print(json.dumps({"mode": mode, "us": {k: round(v, 1) for k, v in sorted(ks.items(), key=lambda t: -t[1])}}))
