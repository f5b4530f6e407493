"""Time k_conv_halo fwd at cfg2 under one FVDB_DEBUG_HALO setting (set in the environment; read once).

FVDB_DEBUG_HALO bits: 1 no MMA, 2 no A build, 4 no output stores, 8 no halo loads, 16 stale weights (k_conv_halo4:
no streamed weight loads or waits at all), 32 no id/record TMAs (ring kernel).  python tools/halo_dbg.py
[cfg2|dense|cfg5|cfg2_32|cfg2_128]  -> one JSON line.  Measured on k_conv_halo4 at cfg2 64x64 (fwd ms): full 0.307,
no streamed weights 0.256, also no MMA 0.223, no MMA + no build 0.187, + no weights 0.140.
"""
import json
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_01781_b200 as P  # noqa: E402
from paper_2407_01781_b200.conv import gather_conv, pack_weights_umma  # noqa: E402
from paper_2407_01781_b200.workloads import sphere_shell_coords  # noqa: E402
from halo_bench import timed  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
C = {"cfg2": 64, "dense": 64, "cfg5": 32, "cfg2_128": 128, "cfg2_32": 32}[cfg]
if cfg == "dense":
    r = np.arange(128)
    coords = np.stack(np.meshgrid(r, r, r, indexing="ij"), -1).reshape(-1, 3)
else:
    coords = sphere_shell_coords(2048 if cfg == "cfg5" else 470, 1.5)
g, _ = P.build_from_coords(coords)
km = P.build_kernel_map(g, g, 1)
x = torch.randn(g.num_voxels, C, device="cuda").to(torch.bfloat16)
w = torch.randn(C, C, 3, 3, 3, device="cuda") / (27 * C) ** 0.5
img = pack_weights_umma(w, False, "halo")
km.fwd.halo_plan(C, C)
t = timed(lambda: gather_conv(x, km.fwd, w, w_image=img, impl="halo"))
print(json.dumps({"cfg": cfg, "dbg": os.environ.get("FVDB_DEBUG_HALO", "0"), "variant": os.environ.get("FVDB_HALO_VARIANT", "-"),
                  "fwd_ms": round(t, 4), "stages_per_sm": round(27 * ((g.num_voxels + 127) // 128) / 148),
                  "cycles_per_stage_at_1.92GHz": round(t * 1e-3 * 1.92e9 / (27 * ((g.num_voxels + 127) // 128) / 148), 1)}))
