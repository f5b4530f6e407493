"""Time the halo-staged vs the gather-GEMM tensor-core conv on a BASELINE config (fwd + dgrad).

python tools/halo_bench.py [cfg2|cfg3|cfg5]  — prints one JSON line per measurement.
Events around single launches, median of 10, 256 MB L2 flush before each launch.
"""
import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2407_01781_b200 as P  # noqa: E402
from paper_2407_01781_b200.conv import gather_conv, pack_weights_umma  # noqa: E402
from paper_2407_01781_b200.workloads import sphere_shell_coords  # noqa: E402


def timed(fn, reps=10):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(3):
        fn()
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
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    import numpy as np
    if cfg.startswith("dense"):  # dense block (100% leaf occupancy): the reference's leaf/brick regime
        side, C = {"dense": (128, 64), "dense128": (96, 128), "dense32": (160, 32)}[cfg]
        r = np.arange(side)
        coords = np.stack(np.meshgrid(r, r, r, indexing="ij"), -1).reshape(-1, 3)
    else:
        res, C = {"cfg2": (470, 64), "cfg5": (2048, 32), "cfg2_128": (470, 128)}[cfg]
        coords = sphere_shell_coords(res, 1.5)
    g, _ = P.build_from_coords(coords)
    km = P.build_kernel_map(g, g, 1)
    n = g.num_voxels
    pairs = km.total_pairs
    x = torch.randn(n, C, device="cuda").to(torch.bfloat16)
    w = torch.randn(C, C, 3, 3, 3, device="cuda") / (27 * C) ** 0.5
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    km.fwd.halo_plan(C, C)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    km.bwd.halo_plan(C, C)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    plan = km.fwd.halo_plan(C, C)
    lv = plan.tensors["tile_level"]
    print(json.dumps({"cfg": cfg, "voxels": n, "pairs": pairs, "plan_fwd_ms": (t1 - t0) * 1e3,
                      "plan_bwd_ms": (t2 - t1) * 1e3, "halo_slots": plan.total_slots,
                      "slots_per_tile": plan.total_slots / lv.numel(),
                      "multi_phase_tiles": int((lv > 1).sum().item())}))
    flop = 2.0 * pairs * C * C
    for impl in ("gather", "halo"):
        imf, imb = pack_weights_umma(w, False, impl), pack_weights_umma(w, True, impl)
        f = timed(lambda: gather_conv(x, km.fwd, w, w_image=imf, impl=impl))
        d = timed(lambda: gather_conv(x, km.bwd, w, transpose=True, w_image=imb, impl=impl))
        print(json.dumps({"impl": impl, "fwd_ms": f, "dgrad_ms": d, "fwd_tflops": flop / f / 1e9,
                          "dgrad_tflops": flop / d / 1e9}))
    yh = gather_conv(x, km.fwd, w, out_dtype=torch.float32, impl="halo")
    yg = gather_conv(x, km.fwd, w, out_dtype=torch.float32, impl="gather")
    print(json.dumps({"max_rel_diff_halo_vs_gather": float((yh - yg).abs().max() / yg.abs().max())}))


if __name__ == "__main__":
    main()
