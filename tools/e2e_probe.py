"""Probe the e2e pipeline: host enqueue time per step vs device time (is there a host sync?)."""
import argparse, json, pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
import bench
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import sphere_shell_coords

g, _ = P.build_from_coords(sphere_shell_coords(470, 1.5))
km = P.build_kernel_map(g, g, 1)
args = argparse.Namespace(e2e_steps=10, steps=10)
# monkeypatch torch.cuda.synchronize counting inside the module path
calls = {"sync": 0}
orig_item = torch.Tensor.item
def item(self):
    calls["sync"] += 1
    return orig_item(self)
torch.Tensor.item = item
t0 = time.perf_counter()
r = bench.run_e2e(args, P, torch, None, g, km, 64, 64, torch.device("cuda"), False)
t1 = time.perf_counter()
print(json.dumps({"e2e_ms": r["ms_per_step"], "wall_s": t1 - t0, "item_calls": calls["sync"]}))
