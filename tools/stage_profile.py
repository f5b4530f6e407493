"""One cfg2 pass of every stage of the path (grid build, kernel map + transpose, first-use gather conv, wgrad)
inside cudaProfilerStart/Stop, for an ncu capture with --profile-from-start off (DRAM bytes per kernel)."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.conv import gather_conv, wgrad
from paper_2407_01781_b200.workloads import sphere_shell_coords
coords = sphere_shell_coords(470, 1.5)
c = torch.from_numpy(coords).cuda()
def run():
    g, _ = P.build_from_coords(c)
    km = P.build_kernel_map(g, g, 1)
    km.bwd
    x = torch.ones(g.num_voxels, 64, device="cuda", dtype=torch.bfloat16)
    w = torch.ones(64, 64, 3, 3, 3, device="cuda") / 1000
    y = gather_conv(x, km.fwd, w, impl="gather")
    wgrad(x, y, km.fwd)
run()
torch.cuda.synchronize()
torch.cuda.profiler.start()
run()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
