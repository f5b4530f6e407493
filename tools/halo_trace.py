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
print("A batches: mma_afull(ab) bld_adone(ab) bld_publish(ab) bload(ab)")
for ab in range(48):
    print(ab, *[int(t[c, ab] - t0) if t[c, ab] else -1 for c in (1, 2, 3, 6)])
print("MMA half0 stages: start(ac) end(ac) | after_bfull(ab) after_afull(ab)")
for a in range(40):
    print(a, *[int(t[c, a] - t0) if t[c, a] else -1 for c in (4, 7)], "|", *[int(t[c, a // 2] - t0) if t[c, a // 2] else -1 for c in (0, 1)])
print("MMA tempty(lt)", [int(t[8, i] - t0) if t[8, i] else -1 for i in range(6)])
print("builder half0 sub0 q0: stage ac: after_loads after_sttm | batch: adone st_waited publish")
for a in range(0, 40, 4):
    ab = a // 2
    print(a, *[int(t[c, a] - t0) if t[c, a] else -1 for c in (4, 7)], "|",
          *[int(t[c, ab] - t0) if t[c, ab] else -1 for c in (2, 8, 3)])
print("phase  ld_hempty ld_idx bld_phase epi_tfull(tile)")
for p in range(10):
    print(p, [(int(t[c, p] - t0) if t[c, p] else -1) for c in (9, 10, 5, 11)])
d = np.diff(t[1, :300])
print(json.dumps({"dbg": os.environ.get("FVDB_DEBUG_HALO"), "mean_cycles_per_A_batch": float(d[d > 0].mean()),
                  "median": float(np.median(d))}))
