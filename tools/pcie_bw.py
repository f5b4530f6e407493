"""Pinned host<->device copy bandwidth: H2D, D2H, and both directions concurrently (GB/s)."""
import json
import torch

n = 256 << 20
h = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(2)]
d = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(2)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def both():
    with torch.cuda.stream(s1):
        d[0].copy_(h[0], non_blocking=True)
    with torch.cuda.stream(s2):
        h[1].copy_(d[1], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t_h2d = timed(lambda: d[0].copy_(h[0], non_blocking=True))
t_d2h = timed(lambda: h[1].copy_(d[1], non_blocking=True))
t_both = timed(both)
print(json.dumps({"h2d_GBps": n / t_h2d / 1e6, "d2h_GBps": n / t_d2h / 1e6,
                  "concurrent_total_GBps": 2 * n / t_both / 1e6, "bytes": n}))
