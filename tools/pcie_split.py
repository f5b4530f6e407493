"""H2D bandwidth of one 130 MB pinned copy vs the same bytes split over 2 / 4 streams (copy engines)."""
import json
import torch

n = 130331648
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]


def run(k):
    step = (n + k - 1) // k
    for i in range(k):
        with torch.cuda.stream(streams[i]):
            d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
    for s in streams[:k]:
        torch.cuda.current_stream().wait_stream(s)


for k in (1, 2, 4):
    run(k)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        run(k)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(json.dumps({"streams": k, "ms": round(ms, 4), "GBps": round(n / ms / 1e6, 1)}))
