import os, time, torch
print("ALLOC_CONF", os.environ.get("PYTORCH_CUDA_ALLOC_CONF"))
x = torch.empty(1, device="cuda")
for n in (110 << 20, 8 << 20, 2 << 20):
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        ts.append((time.perf_counter() - t0) * 1e6)
        del t
    print(n >> 20, "MB alloc us:", [round(v) for v in ts])
keep = []
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    keep.append(torch.empty(110 << 20, dtype=torch.uint8, device="cuda"))
    ts.append((time.perf_counter() - t0) * 1e6)
print("held allocs us", [round(v) for v in ts])
print(torch.cuda.memory_stats()["num_alloc_retries"], torch.cuda.memory_stats()["segment.all.allocated"])
