"""Time k_wgrad_tc on cfg2 under FVDB_DEBUG_WG switches (1 no MMA, 2 no A gather); CH env = channels."""
import json, os, subprocess, sys, pathlib
if len(sys.argv) > 1 and sys.argv[1] == "run":
    sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
    import torch
    import paper_2407_01781_b200 as P
    from paper_2407_01781_b200.conv import wgrad
    from paper_2407_01781_b200.workloads import sphere_shell_coords
    g, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
    km = P.build_kernel_map(g, g, 1)
    ch = int(os.environ.get("CH", "64"))  # channels (Cin = Cout)
    x = torch.randn(g.num_voxels, ch, device="cuda").to(torch.bfloat16)
    gy = torch.randn(g.num_voxels, ch, device="cuda").to(torch.bfloat16)
    for _ in range(3):
        wgrad(x, gy, km.fwd)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); wgrad(x, gy, km.fwd); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(json.dumps({"dbg": os.environ.get("FVDB_DEBUG_WG", "0"), "ms": sorted(ts)[len(ts) // 2]}))
else:
    for d in sys.argv[1:] or ("0", "1", "2", "3"):
        r = subprocess.run([sys.executable, __file__, "run"], env={**os.environ, "FVDB_DEBUG_WG": d},
                           capture_output=True, text=True, timeout=120)
        print(r.stdout.strip() or r.stderr[-400:])
