"""k_conv_halo2 timeline (cluster 0, set 0) from the FVDB_DEBUG_HALO=64 trace, cfg2 64x64.
Clocks of the two CTAs are per-SM counters: only same-CTA differences are meaningful, except channel 5 (rank-1
builder) which is compared with itself."""
import ctypes as C, json, os, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
os.environ.setdefault("FVDB_DEBUG_HALO", "64")
import numpy as np, torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200 import _lib
from paper_2407_01781_b200.conv import gather_conv, pack_weights_umma
from paper_2407_01781_b200.workloads import sphere_shell_coords
g, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
km = P.build_kernel_map(g, g, 1)
x = torch.randn(g.num_voxels, 64, device="cuda").to(torch.bfloat16)
w = torch.randn(64, 64, 3, 3, 3, device="cuda") / (27 * 64) ** 0.5
img = pack_weights_umma(w, False, "halo")
for _ in range(3):
    gather_conv(x, km.fwd, w, w_image=img, impl="halo")
torch.cuda.synchronize()
L = _lib.lib()
L.fvdb_halo_debug_trace.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(12 * 2048, np.int64)
_lib.check(L.fvdb_halo_debug_trace(buf.ctypes.data, buf.size), "trace")
t = buf.reshape(12, 2048)
lo, hi = 20, 220
d = lambda a, b: float(np.median(t[a, lo:hi] - t[b, lo:hi]))
print(json.dumps({
    "b0_afree_wait": d(0, 7), "b0_build": d(1, 0), "b0_period": float(np.median(np.diff(t[7, lo:hi]))),
    "b1_period": float(np.median(np.diff(t[5, lo:hi]))),
    "iss_bar_after_b0_arrive": d(2, 1), "iss_pfull_wait": d(3, 2), "iss_dempty_wait": d(6, 3),
    "iss_issue_commit": d(4, 6), "iss_period": float(np.median(np.diff(t[2, lo:hi]))),
    "afree_after_commit_js-2": float(np.median(t[0, lo + 2:hi + 2] - t[4, lo:hi])),
}))
