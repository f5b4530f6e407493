"""Per-stage timeline of k_conv_halo4 (CTA 0, set 0) from the FVDB_DEBUG_HALO=64 trace (cfg2 64->64).

Channels: 7 stage start, 0 after A-slot wait, 1 after build + wait::st, 2 after the set barrier, 3 after the
weight / accumulator waits, 4 after MMA issue + commits; 5 weight loader TMA issue (set 0); 6 epilogue D_0
ready; 8 halo loader phase start; 9 / 10 set 0 before / after the phase's halo + record waits.
"""
import ctypes as C, json, os, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
os.environ.setdefault("FVDB_DEBUG_HALO", "64")
import numpy as np, torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200 import _lib
from paper_2407_01781_b200.conv import gather_conv, pack_weights_umma
from paper_2407_01781_b200.workloads import sphere_shell_coords
CH = int(os.environ.get("CH", "64"))
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
_lib.check(L.fvdb_halo_debug_trace(buf.ctypes.data, buf.size), "trace")
t = buf.reshape(12, 2048)
n = 200
lo, hi = 20, 20 + n
st = t[7, lo:hi]
out = {}
d = lambda c1, c0, sh=0: float(np.median(t[c1, lo + sh:hi + sh] - t[c0, lo:hi]))
out["builder_afree_wait"] = d(0, 7)
out["builder_build"] = d(1, 0)
out["builder_period"] = float(np.median(np.diff(t[7, lo:hi])))
out["issuer_barrier_after_builder_arrive"] = d(2, 1)
out["issuer_waits"] = d(3, 2)
out["issuer_issue_commit"] = d(4, 3)
out["issuer_period"] = float(np.median(np.diff(t[2, lo:hi])))
out["wload_issue_minus_stage_start"] = d(5, 7)
out["tma_issue_to_issuer_past_waits"] = d(3, 5)
out["loader_poll_start_to_issue"] = d(5, 11)
out["commit_j-3_to_poll_start_j"] = float(np.median(t[11, lo + 3:hi + 3] - t[4, lo:hi]))
out["commit_j_to_builder_afree_j+2"] = float(np.median(t[0, lo + 2:hi + 2] - t[4, lo:hi]))
out["commit_j-3_to_tma_issue_j"] = float(np.median(t[5, lo + 3:hi + 3] - t[4, lo:hi]))
ph = t[9, 5:60]
out["phase_wait"] = float(np.median(t[10, 5:60] - t[9, 5:60]))
out["epi_tile_period"] = float(np.median(np.diff(t[6, 5:60])))
out["loader_phase_period"] = float(np.median(np.diff(t[8, 5:60])))
print(json.dumps(out))
# loader: 5 phase top, 8 after the id / buffer waits, 11 after the cp.async loop
ld = {"loader_top_to_after_waits": float(np.median(t[8, 5:60] - t[5, 5:60])),
      "loader_cp_async_loop": float(np.median(t[11, 5:60] - t[8, 5:60])),
      "loader_after_loop_to_next_top": float(np.median(t[5, 6:61] - t[11, 5:60]))}
print(json.dumps(ld))
