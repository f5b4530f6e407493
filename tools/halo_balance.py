"""Per-CTA start/end times of k_conv_halo (FVDB_DEBUG_HALO=128): how evenly the static round-robin tile
assignment spreads the work. python tools/halo_balance.py [cfg2|cfg5|lidar] -> one JSON line."""
import ctypes as C, json, os, pathlib, sys
os.environ["FVDB_DEBUG_HALO"] = "128"
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch  # noqa: E402
import paper_2407_01781_b200 as P  # noqa: E402
from paper_2407_01781_b200 import _lib  # noqa: E402
from paper_2407_01781_b200.conv import gather_conv, pack_weights_umma  # noqa: E402
from paper_2407_01781_b200.workloads import sphere_shell_coords  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
CH = 32 if cfg == "cfg5" else 64
if cfg == "lidar":
    from paper_2407_01781_b200.workloads import lidar_scan_points
    g, _ = P.build_from_points(lidar_scan_points(0), P.VoxelTransform.uniform(0.05))
else:
    g, _ = P.build_from_coords(sphere_shell_coords(2048 if cfg == "cfg5" else 470, 1.5))
km = P.build_kernel_map(g, g, 1)
x = torch.randn(g.num_voxels, CH, device="cuda").to(torch.bfloat16)
w = torch.randn(CH, CH, 3, 3, 3, device="cuda") / (27 * CH) ** 0.5
img = pack_weights_umma(w, False, "halo")
for _ in range(3):
    gather_conv(x, km.fwd, w, w_image=img, impl="halo")
torch.cuda.synchronize()
L = _lib.lib()
L.fvdb_halo_debug_cta.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(1024 * 2, np.int64)
L.fvdb_halo_debug_cta(buf.ctypes.data, buf.size)
t = buf.reshape(1024, 2)
t = t[t[:, 1] > 0]
t0 = t[:, 0].min()
start, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
dur = end - start
print(json.dumps({"cfg": cfg, "ctas": len(t), "tiles": int((g.num_voxels + 127) // 128),
                  "kernel_us": float(end.max()), "cta_us_min": float(dur.min()), "cta_us_median": float(np.median(dur)),
                  "cta_us_max": float(dur.max()), "start_spread_us": float(start.max()),
                  "end_p10_us": float(np.percentile(end, 10)), "idle_frac": float(1 - dur.sum() / (len(t) * end.max()))}))
