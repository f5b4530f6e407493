"""Time k_conv_halo on cfg2 under FVDB_DEBUG_HALO switches (1 no MMA, 2 no A build, 4 no stores, 8 no halo loads)."""
import json, os, subprocess, sys, pathlib
if len(sys.argv) > 1 and sys.argv[1] == "run":  # child
    sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
    import torch
    import paper_2407_01781_b200 as P
    from paper_2407_01781_b200.conv import gather_conv, pack_weights_umma
    from paper_2407_01781_b200.workloads import sphere_shell_coords
    g, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
    km = P.build_kernel_map(g, g, 1)
    x = torch.randn(g.num_voxels, 64, device="cuda").to(torch.bfloat16)
    w = torch.randn(64, 64, 3, 3, 3, device="cuda") / 40
    img = pack_weights_umma(w, False, "halo")
    km.fwd.halo_plan(64, 64)
    for _ in range(3):
        gather_conv(x, km.fwd, w, w_image=img, impl="halo")
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); gather_conv(x, km.fwd, w, w_image=img, impl="halo"); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(json.dumps({"dbg": os.environ.get("FVDB_DEBUG_HALO", "0"), "ms": sorted(ts)[len(ts) // 2]}))
else:
    for d in sys.argv[1:] or ("0", "16", "31", "15", "17"):
        r = subprocess.run([sys.executable, __file__, "run"], env={**os.environ, "FVDB_DEBUG_HALO": d},
                           capture_output=True, text=True, timeout=120)
        print(r.stdout.strip() or r.stderr[-400:])
