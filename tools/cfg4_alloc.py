"""cfg4 step wall time per 20-step loop with caching-allocator statistics (new device segments = cudaMalloc)."""
import pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import sphere_shell_coords
coords = sphere_shell_coords(470, 1.5)
pts = torch.from_numpy(coords.astype(np.float64)).cuda()
tf = P.VoxelTransform.uniform(1.0)
down = P.SparseConv3d(64, 128, stride=2).cuda()
up = P.SparseConv3d(128, 64, stride=2, transposed=True).cuda()
x = torch.randn(coords.shape[0], 64, device="cuda")
import os
if os.environ.get("PRIME"):  # reserve one large cached segment up front; later allocations split it
    torch.empty(int(os.environ["PRIME"]) << 30, dtype=torch.uint8, device="cuda")
def step():
    g, _ = P.build_from_points(pts, tf)
    fine = P.GridBatch([g])
    coarse, h = down(fine, fine.jagged(x))
    _, y = up(coarse, h, out_grid=fine)
    y.jdata.sum(dtype=torch.float32).backward()
for loop in range(4):
    s0 = torch.cuda.memory_stats()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(20):
        step()
    torch.cuda.synchronize(); t1 = time.perf_counter()
    s1 = torch.cuda.memory_stats()
    print(f"loop {loop}: {(t1 - t0) / 20 * 1e3:.2f} ms/step, new segments "
          f"{s1['segment.all.allocated'] - s0['segment.all.allocated']}, frees {s1['segment.all.freed'] - s0['segment.all.freed']}, "
          f"retries {s1['num_alloc_retries'] - s0['num_alloc_retries']}, reserved {s1['reserved_bytes.all.current'] / 2**30:.2f} GiB")
