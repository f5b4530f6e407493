import sys, pathlib
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import sphere_shell_coords
from paper_2407_01781_b200.conv import HaloPlan
g, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
km = P.build_kernel_map(g, g, 1)
for cap in (440, 400, 360, 320, 300):
    p = HaloPlan(km.fwd, cap)
    lv = p.tensors["tile_level"].cpu().numpy(); ph = p.tensors["phase"].cpu().numpy()
    l1 = ph[lv == 1, 0, 1]
    print(cap, "multi-phase tiles", int((lv > 1).sum()), "of", len(lv), "len pcts", np.percentile(l1, [50, 90, 99, 100]).tolist())
