"""Halo kernel fwd time at cfg2 64x64 with plans built for a smaller phase capacity (more multi-phase tiles):
separates the multi-phase penalty from other changes that shrink the capacity (e.g. more weight slots)."""
import json, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200 import _lib
from paper_2407_01781_b200.conv import HaloPlan, gather_conv, pack_weights_umma
from paper_2407_01781_b200.workloads import sphere_shell_coords
from halo_bench import timed
g, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
km = P.build_kernel_map(g, g, 1)
x = torch.randn(g.num_voxels, 64, device="cuda").to(torch.bfloat16)
w = torch.randn(64, 64, 3, 3, 3, device="cuda") / (27 * 64) ** 0.5
img = pack_weights_umma(w, False, "halo")
kcap = int(_lib.lib().fvdb_halo_cap(64, 64))
for cap in [c for c in (440, 400, 368, 340, 312) if c <= kcap]:
    km.fwd._plans[kcap] = HaloPlan(km.fwd, cap)
    t = timed(lambda: gather_conv(x, km.fwd, w, w_image=img, impl="halo"))
    lv = km.fwd._plans[kcap].tensors["tile_level"]
    print(json.dumps({"plan_cap": cap, "kernel_cap": kcap, "multi_phase_tiles": int((lv > 1).sum()), "fwd_ms": round(t, 4)}))
