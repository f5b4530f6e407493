"""Device time of the kernel-map kernels (torch.profiler) for cfg2 (stride 1) and cfg4 (stride 2)."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import sphere_shell_coords
g, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
gc = P.coarsen(g, 2)
for gi, go, s in ((g, g, 1), (g, gc, 2)):
    for _ in range(3):
        P.build_kernel_map(gi, go, s)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            P.build_kernel_map(gi, go, s)
        torch.cuda.synchronize()
    for e in prof.key_averages():
        if e.device_time_total > 0:
            print(f"stride {s}: {e.key[:60]:60s} {e.device_time_total / e.count:9.1f} us x{e.count}")
