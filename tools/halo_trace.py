"""Pipeline trace of k_conv_halo (CTA 0) on cfg2: FVDB_DEBUG_HALO=64 (+ other switch bits)."""
import ctypes as C, json, os, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200 import _lib
from paper_2407_01781_b200.conv import gather_conv, pack_weights_umma
from paper_2407_01781_b200.workloads import sphere_shell_coords
g, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
km = P.build_kernel_map(g, g, 1)
x = torch.randn(g.num_voxels, 64, device="cuda").to(torch.bfloat16)
w = torch.randn(64, 64, 3, 3, 3, device="cuda") / 40
img = pack_weights_umma(w, False, "halo")
for _ in range(3):
    gather_conv(x, km.fwd, w, w_image=img, impl="halo")
torch.cuda.synchronize()
L = _lib.lib()
L.fvdb_halo_debug_trace.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(12 * 2048, np.int64)
L.fvdb_halo_debug_trace(buf.ctypes.data, buf.size)
t = buf.reshape(12, 2048)
t0 = t[t > 0].min()
t = t.astype(np.int64)
def col(ch, n):
    return [int(t[ch, i] - t0) if t[ch, i] else -1 for i in range(n)]
print("A batches: mma_afull(ab) bld_adone(ab) bld_publish(ab)")
for ab in range(40):
    print(ab, int(t[1, ab] - t0) if t[1, ab] else -1, int(t[2, ab] - t0) if t[2, ab] else -1,
          int(t[3, ab] - t0) if t[3, ab] else -1)
print("MMA stages: start(ac) before_commit(ac)")
for a in range(60):
    print(a, int(t[4, a] - t0) if t[4, a] else -1, int(t[7, a] - t0) if t[7, a] else -1)
print("B batches: mma_bfull(bb) bload(bb)")
for bb in range(20):
    print(bb, int(t[0, bb] - t0) if t[0, bb] else -1, int(t[6, bb] - t0) if t[6, bb] else -1)
print("phase  ld_xfull ld_hempty ld_idx bld_phase epi_tfull")
for p in range(8):
    print(p, [(int(t[c, p] - t0) if t[c, p] else -1) for c in (8, 9, 10, 5, 11)])
d = np.diff(t[1, :300])
print(json.dumps({"dbg": os.environ.get("FVDB_DEBUG_HALO"), "mean_cycles_per_A_batch": float(d[d > 0].mean()),
                  "median": float(np.median(d))}))
