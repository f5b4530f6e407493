"""Slot round-trip analysis of k_conv_halo (CTA 0, cfg2 64->64) from the FVDB_DEBUG_HALO=64 trace.

Channels (csrc/conv_halo.cu trace points): 0 MMA after BFULL(ab), 1 MMA after AFULL(ab), 2 builder after
ADONE(ab), 3 builder publish(ab), 6 weight loader after ADONE(ab), 9 loader phase start, 11 epilogue tfull.
Per batch ab (half ab&1, slot reuse every 2*NSL batches) prints median cycle intervals over a window.
"""
import ctypes as C, json, os, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200 import _lib
from paper_2407_01781_b200.conv import gather_conv, pack_weights_umma
from paper_2407_01781_b200.workloads import sphere_shell_coords
NSL = int(os.environ.get("NSL", "2"))  # per-half slots (two-issuer layout); R overrides the reuse distance
CH = int(os.environ.get("CH", "64"))  # channels (K = N); CFG=dense uses a 160^3 block instead of the cfg2 shell
if os.environ.get("CFG") == "dense":
    r = np.arange(160)
    g, _ = P.build_from_coords(np.stack(np.meshgrid(r, r, r, indexing="ij"), -1).reshape(-1, 3))
else:
    g, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
km = P.build_kernel_map(g, g, 1)
x = torch.randn(g.num_voxels, CH, device="cuda").to(torch.bfloat16)
w = torch.randn(CH, CH, 3, 3, 3, device="cuda") / (27 * CH) ** 0.5
img = pack_weights_umma(w, False, "halo")
for _ in range(3):
    gather_conv(x, km.fwd, w, w_image=img, impl="halo")
torch.cuda.synchronize()
L = _lib.lib()
L.fvdb_halo_debug_trace.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(12 * 2048, np.int64)
L.fvdb_halo_debug_trace(buf.ctypes.data, buf.size)
t = buf.reshape(12, 2048).astype(np.int64)
lo, hi = 100, 300
ab = np.arange(lo, hi)
R = int(os.environ.get("R", str(2 * NSL)))  # batches between two uses of one slot
def med(a):
    a = a[(a > -10**7) & (a < 10**7)]
    return float(np.median(a)) if a.size else None
out = {
    "dbg": os.environ.get("FVDB_DEBUG_HALO"),
    "mma_batch_interval(ch1[ab+2]-ch1[ab])": med(t[1, ab + 2] - t[1, ab]),
    "slot_round_trip(ch1[ab]-ch1[ab-R])": med(t[1, ab] - t[1, ab - R]),
    "commit_to_builder_wake(ch2[ab]-ch1[ab-R])": med(t[2, ab] - t[1, ab - R]),
    "build(ch3[ab]-ch2[ab])": med(t[3, ab] - t[2, ab]),
    "publish_to_mma(ch1[ab]-ch3[ab])": med(t[1, ab] - t[3, ab]),
    "mma_wait_afull_after_bfull(ch1-ch0)": med(t[1, ab] - t[0, ab]),
    "commit_to_bload_wake(ch6[ab]-ch1[ab-R])": med(t[6, ab] - t[1, ab - R]),
    "weight_tma(ch0[ab]-ch6[ab])": med(t[0, ab] - t[6, ab]),
    "tile_interval(ch11)": med(np.diff(t[11, 5:40])),
    "loader_issue(ch10[p]-ch9[p])": med(t[10, 5:60] - t[9, 5:60]),
    "loader_wait_hempty(ch9[p+1]-ch10[p])": med(t[9, 6:61] - t[10, 5:60]),
    "builder_phase_start_after_record(ch5[p]-ch10[p])": med(t[5, 5:60] - t[10, 5:60]),
    "phase_interval(ch9)": med(np.diff(t[9, 5:60])),
}
print(json.dumps(out))
