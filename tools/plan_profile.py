"""Per-kernel device time of one halo-plan build (cfg2 shell, 64x64, fresh transposed table)."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import sphere_shell_coords
g, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
for rep in range(2):
    km = P.build_kernel_map(g, g, 1)
    t = km.bwd
    t.colors()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        t.halo_plan(64, 64)
        torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12, max_name_column_width=50))
