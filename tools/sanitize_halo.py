"""Small halo / wgrad launches for compute-sanitizer (racecheck, synccheck): one forward and one transposed per
(K, N), the table and pair-list wgrad.  compute-sanitizer --tool racecheck python tools/sanitize_halo.py"""
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2407_01781_b200 as P  # noqa: E402
from paper_2407_01781_b200.workloads import sphere_shell_coords  # noqa: E402

CONV = sys.modules["paper_2407_01781_b200.conv"]
g, _ = P.build_from_coords(sphere_shell_coords(24, band=1.5))
km = P.build_kernel_map(g, g, 1)
n = g.num_voxels
for K, N in [(64, 64), (32, 32), (128, 128)]:
    x = torch.randn(n, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(N, K, 3, 3, 3, device="cuda") / (27 * K) ** 0.5
    gy = torch.randn(n, N, device="cuda").to(torch.bfloat16)
    CONV.gather_conv(x, km.fwd, w, out_dtype=torch.float32, impl="halo")
    CONV.gather_conv(gy, km.bwd, w, transpose=True, out_dtype=torch.float32, impl="halo")
    CONV.wgrad(x, gy, km.fwd)
os.environ["FVDB_WG_PAIRS"] = "force"
x = torch.randn(n, 128, device="cuda").to(torch.bfloat16)
CONV.wgrad(x, x, km.fwd)
torch.cuda.synchronize()
print("sanitize run done", n)
