"""Stress the halo conv: rerun it (fixed plan and inputs) many times against the gather kernel and characterise
any wrong output rows (tiles, rows within the tile, channels).

python tools/halo_stress.py RUNS [C=64|32] [fwd|bwd]  -> JSON lines (first three failures, then a summary).
Found the two-loader-warp row-id race in k_conv_halo4 (2 of 300 cfg2 forwards wrong, all in tile 2: the
plan's first multi-phase tile, CTA 2's first tile); 0 of 600 after the xempty barrier.
"""
import os, sys, pathlib, json, collections
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.conv import gather_conv
from paper_2407_01781_b200.workloads import sphere_shell_coords
C = int(sys.argv[2]) if len(sys.argv) > 2 else 64
c = sphere_shell_coords(2048 if C == 32 else 470, band=1.5)
g, _ = P.build_from_coords(c)
km = P.build_kernel_map(g, g, 1)
n = g.num_voxels
gen = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(n, C, device="cuda", generator=gen).to(torch.bfloat16)
w = torch.randn(C, C, 3, 3, 3, device="cuda", generator=gen) / (27 * C) ** 0.5
ref = gather_conv(x, km.fwd, w, out_dtype=torch.float32, impl="gather")
mode = sys.argv[3] if len(sys.argv) > 3 else "fwd"
tab = km.fwd if mode == "fwd" else km.bwd
if mode != "fwd":
    ref = gather_conv(x, km.bwd, w, transpose=True, out_dtype=torch.float32, impl="gather")
runs = int(sys.argv[1]) if len(sys.argv) > 1 else 100
fails = 0
rowpos = collections.Counter(); colpat = collections.Counter(); nbad = []
tol = 1e-3 * float(ref.abs().max())
for it in range(runs):
    y = gather_conv(x, tab, w, transpose=(mode != "fwd"), out_dtype=torch.float32, impl="halo")
    d = (y - ref).abs()
    badr = (d.amax(1) > tol).nonzero().squeeze(1)
    if len(badr):
        fails += 1
        nbad.append(len(badr))
        for r in badr[:64].tolist():
            rowpos[r % 128] += 1
        bc = (d[badr] > tol)
        colpat[str(bc.sum(1)[:8].tolist())] += 1
        if fails <= 3:
            r0 = int(badr[0])
            print(json.dumps({"it": it, "bad_rows": len(badr), "rows": badr[:12].tolist(),
                              "tiles": sorted(set((badr // 128).tolist()))[:10],
                              "bad_cols_first_row": (d[r0] > tol).nonzero().squeeze(1).tolist()[:64],
                              "got": y[r0, :4].tolist(), "want": ref[r0, :4].tolist()}))
print(json.dumps({"C": C, "mode": mode, "runs": runs, "fails": fails, "nbad": nbad[:20],
                  "rowpos_top": rowpos.most_common(12), "colpat": colpat.most_common(5)}))
