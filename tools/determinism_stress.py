"""Bitwise repeatability of every hot kernel: each case runs RUNS times on fixed inputs and must reproduce its
first result exactly (all kernels here are deterministic by design).  A data race between warps shows up as
an occasional mismatch (tools/halo_stress.py characterises the halo kernels' wrong rows).

python tools/determinism_stress.py [RUNS=50]  -> one JSON line per case + a summary line.
"""
import json
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2407_01781_b200 as P  # noqa: E402
from paper_2407_01781_b200.workloads import lidar_scan_points, sphere_shell_coords  # noqa: E402

CONV = sys.modules["paper_2407_01781_b200.conv"]
RUNS = int(sys.argv[1]) if len(sys.argv) > 1 else 50
gen = torch.Generator(device="cuda").manual_seed(11)
shell = sphere_shell_coords(470, band=1.5)
g, _ = P.build_from_coords(shell)
km = P.build_kernel_map(g, g, 1)
lid, _ = P.build_from_points(P.jagged_from_list([torch.from_numpy(lidar_scan_points(s)) for s in range(2)]),
                             P.VoxelTransform.uniform(0.05))
kml = P.build_batch_kernel_map(lid, lid, 1)
n, nl = g.num_voxels, lid.total_voxels


def feats(rows, c):
    return torch.randn(rows, c, device="cuda", generator=gen).to(torch.bfloat16)


def weights(co, ci):
    return torch.randn(co, ci, 3, 3, 3, device="cuda", generator=gen) / (27 * ci) ** 0.5


cases = {}
for K, N in [(64, 64), (32, 32), (32, 64), (64, 32), (128, 128)]:
    x, w = feats(n, K), weights(N, K)
    cases[f"halo_fwd_{K}x{N}"] = (lambda x=x, w=w: CONV.gather_conv(x, km.fwd, w, out_dtype=torch.float32, impl="halo"))
    gy = feats(n, N)
    cases[f"halo_dgrad_{K}x{N}"] = (lambda gy=gy, w=w: CONV.gather_conv(gy, km.bwd, w, transpose=True,
                                                                      out_dtype=torch.float32, impl="halo"))
x64, w64, gy64 = feats(n, 64), weights(64, 64), feats(n, 64)
cases["gather_fwd_64x64"] = lambda: CONV.gather_conv(x64, km.fwd, w64, out_dtype=torch.float32, impl="gather")
cases["wgrad_table_64x64"] = lambda: CONV.wgrad(x64, gy64, km.fwd)
xl, wl, gyl = feats(nl, 128), weights(128, 128), feats(nl, 128)


def sorted_gather():
    os.environ["FVDB_SIG_SORT"] = "force"
    try:
        return CONV.gather_conv(xl, kml.fwd, wl, out_dtype=torch.float32, impl="gather")
    finally:
        del os.environ["FVDB_SIG_SORT"]


cases["sorted_gather_lidar_128"] = sorted_gather


def wgrad_pairs(sched):
    def f():
        os.environ["FVDB_WG_PAIRS"] = "force"
        old, CONV._WG_PAIRS_SCHED = CONV._WG_PAIRS_SCHED, sched
        try:
            return CONV.wgrad(xl, gyl, kml.fwd)
        finally:
            CONV._WG_PAIRS_SCHED = old
            del os.environ["FVDB_WG_PAIRS"]
    return f


cases["wgrad_pairs_linear_lidar"] = wgrad_pairs("linear")
cases["wgrad_pairs_tiles_lidar"] = wgrad_pairs("tiles")
cases["kernel_map_cfg2"] = lambda: P.build_kernel_map(g, g, 1).nbr
cases["grid_build_cfg2"] = lambda: P.build_from_coords(shell)[0].leaf_masks

summary = {}
for name, fn in cases.items():
    try:
        first = fn()
        torch.cuda.synchronize()
        bad = 0
        for _ in range(RUNS):
            bad += int(not torch.equal(fn(), first))
        summary[name] = bad
        print(json.dumps({"case": name, "runs": RUNS, "mismatches": bad}), flush=True)
    except Exception as e:  # noqa: BLE001
        summary[name] = f"error: {e}"[:120]
        print(json.dumps({"case": name, "error": str(e)[:200]}), flush=True)
print(json.dumps({"summary": summary}))
