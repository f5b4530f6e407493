"""Time k_conv_fwd_tc on cfg2 with profiling switches (FVDB_DEBUG_FWD: 1 = no MMA, 2 = no stores)."""
import json, os, subprocess, sys
if len(sys.argv) > 1:
    import pathlib
    sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
    import torch
    import paper_2407_01781_b200 as P
    from paper_2407_01781_b200.conv import gather_conv, pack_weights_umma
    from paper_2407_01781_b200.workloads import sphere_shell_coords
    g, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
    km = P.build_kernel_map(g, g, 1)
    x = torch.randn(g.num_voxels, 64, device="cuda").to(torch.bfloat16)
    w = torch.randn(64, 64, 3, 3, 3, device="cuda") / 40
    img = pack_weights_umma(w, False)
    for _ in range(3):
        gather_conv(x, km.fwd, w, w_image=img)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); gather_conv(x, km.fwd, w, w_image=img); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(json.dumps({"dbg": os.environ.get("FVDB_DEBUG_FWD", "0"), "ms": sorted(ts)[len(ts) // 2]}))
else:
    for npw in ("4", "8"):
        for d in ("0", "1"):
            r = subprocess.run([sys.executable, __file__, "run"], env={**os.environ, "FVDB_DEBUG_FWD": d,
                               "FVDB_FWD_NPW": npw}, capture_output=True, text=True)
            print("npw", npw, r.stdout.strip() or r.stderr[-500:])
