"""Weight gradient over the neighbour table (fvdb_conv_wgrad_tc) vs over per-offset pair lists
(fvdb_conv_wgrad_pairs_tc), per map and channel shape: median of 10 event-timed launches with a 256 MB L2
flush before each, the one-off pair-list build, and the relative difference of the two results.
python tools/wgrad_pairs_bench.py -> one JSON line per case."""
import json, os, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import paper_2407_01781_b200 as P  # noqa: E402
from paper_2407_01781_b200.conv import wgrad  # noqa: E402
from paper_2407_01781_b200.workloads import sphere_shell_coords, lidar_scan_points  # noqa: E402


def timed(fn, reps=10):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def main():
    g, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
    gc = P.coarsen(g, 2)
    km2 = P.build_kernel_map(g, gc, 2)
    km1 = P.build_kernel_map(g, g, 1)
    g3, _ = P.build_from_points(lidar_scan_points(0), P.VoxelTransform.uniform(0.05))
    km3 = P.build_kernel_map(g3, g3, 1)
    cases = [("cfg3_lidar", km3.fwd, g3.num_voxels, 128, 128),
             ("lidar_64x128", km3.fwd, g3.num_voxels, 64, 128),
             ("lidar_128x64", km3.fwd, g3.num_voxels, 128, 64),
             ("cfg4_s2_64x128", km2.fwd, g.num_voxels, 64, 128),
             ("cfg4_s2_128x64", km2.fwd, g.num_voxels, 128, 64),
             ("shell_s1_128x128", km1.fwd, g.num_voxels, 128, 128),
             ("shell_s1_64x128", km1.fwd, g.num_voxels, 64, 128)]
    for name, tab, n_in, cin, cout in cases:
        x = torch.randn(n_in, cin, device="cuda").to(torch.bfloat16)
        go = torch.randn(tab.n, cout, device="cuda").to(torch.bfloat16)
        tab._pairs = None
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); tab.pair_lists(); b.record(); torch.cuda.synchronize()
        build_ms = a.elapsed_time(b)
        res = {}
        for mode in ("0", "force"):
            os.environ["FVDB_WG_PAIRS"] = mode
            res[mode] = timed(lambda: wgrad(x, go, tab))
        os.environ["FVDB_WG_PAIRS"] = "0"
        r0 = wgrad(x, go, tab)
        os.environ["FVDB_WG_PAIRS"] = "force"
        r1 = wgrad(x, go, tab)
        r2 = wgrad(x, go, tab)
        rel = float((r0 - r1).abs().max() / r0.abs().max())
        print(json.dumps({"case": name, "rows": tab.n, "density": round(tab.density(), 2), "table_ms": res["0"],
                          "pairs_ms": res["force"], "pair_lists_ms": build_ms, "rel_diff": rel,
                          "deterministic": bool(torch.equal(r1, r2))}), flush=True)


if __name__ == "__main__":
    main()
