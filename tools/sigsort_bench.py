"""Gather-GEMM conv over signature-sorted vs unsorted tables (cfg4 stride-2 maps, cfg2 stride-1 map).

python tools/sigsort_bench.py (GRID=1: more shapes; SKIP_HALO=1: gather only) — one JSON line per (map, mode): median of 10 event-timed launches,
256 MB L2 flush before each; plus the one-off cost of fvdb_kmap_signature_order.
"""
import json
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2407_01781_b200 as P  # noqa: E402
from paper_2407_01781_b200.conv import gather_conv, pack_weights_umma  # noqa: E402
from paper_2407_01781_b200.workloads import sphere_shell_coords  # noqa: E402


def timed(fn, reps=10):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def main():
    g, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
    gc = P.coarsen(g, 2)
    km2 = P.build_kernel_map(g, gc, 2)
    km1 = P.build_kernel_map(g, g, 1)
    from paper_2407_01781_b200.workloads import lidar_scan_points
    g3, _ = P.build_from_points(lidar_scan_points(0), P.VoxelTransform.uniform(0.05))
    km3 = P.build_kernel_map(g3, g3, 1)
    import os as _os
    if _os.environ.get("GRID") == "1":  # density x channel-width grid for the conv-kernel policy
        cases = [(f"shell_s1_{k}x{n}", km1.fwd, k, n, False, g.num_voxels) for k, n in ((128, 128), (64, 128), (128, 64), (32, 32), (32, 64))]
        cases += [(f"lidar_s1_{k}x{n}", km3.fwd, k, n, False, g3.num_voxels) for k, n in ((64, 64), (32, 32), (64, 128))]
    else:
        cases = []
    cases += [("cfg3_lidar_fwd", km3.fwd, 128, 128, False, g3.num_voxels),
             ("cfg4_down_fwd", km2.fwd, 64, 128, False, g.num_voxels),
             ("cfg4_up_T", km2.bwd, 128, 64, True, gc.num_voxels),
             ("cfg2_s1", km1.fwd, 64, 64, False, g.num_voxels)]
    for name, tab, K, N, tr, n_in in cases:
        x = torch.randn(n_in, K, device="cuda").to(torch.bfloat16)
        w = torch.randn(*((K, N) if tr else (N, K)), 3, 3, 3, device="cuda") / (27 * K) ** 0.5
        img = pack_weights_umma(w, tr, "gather")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tab._sorted = None
        a.record()
        tab.signature_sorted()
        b.record()
        torch.cuda.synchronize()
        sort_ms = a.elapsed_time(b)
        tab._sorted = None
        sort_ms = min(sort_ms, timed(lambda: (setattr(tab, "_sorted", None), tab.signature_sorted()), 5))
        res = {}
        for on in ("0", "force"):
            os.environ["FVDB_SIG_SORT"] = on
            res[on] = timed(lambda: gather_conv(x, tab, w, transpose=tr, w_image=img))
        halo = None
        if not os.environ.get("SKIP_HALO"):
            imh = pack_weights_umma(w, tr, "halo")
            tab.halo_plan(K, N)
            halo = timed(lambda: gather_conv(x, tab, w, transpose=tr, w_image=imh))
        print(json.dumps({"map": name, "rows": tab.n, "density": round(tab.density(), 2), "unsorted_ms": res["0"],
                          "sorted_ms": res["force"], "sort_ms": sort_ms, "halo_ms": halo}))


if __name__ == "__main__":
    main()
