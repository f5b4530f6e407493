"""cfg5 weight gradient on the halo plan (fvdb_conv_wgrad_halo) for an ncu capture."""
import os, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
os.environ["FVDB_WG_HALO"] = "force"
import torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.conv import wgrad
from paper_2407_01781_b200.workloads import sphere_shell_coords
g, _ = P.build_from_coords(sphere_shell_coords(2048 if (sys.argv[1:] or ["cfg5"])[0] == "cfg5" else 470, 1.5))
km = P.build_kernel_map(g, g, 1)
x = torch.randn(g.num_voxels, 32, device="cuda").to(torch.bfloat16)
gy = torch.randn(g.num_voxels, 32, device="cuda").to(torch.bfloat16)
for _ in range(3):
    wgrad(x, gy, km.fwd)
torch.cuda.synchronize()
