"""H2D bandwidth probe: 2 x 12 MB pinned -> device, one stream vs two concurrent streams."""
import time
import torch
n = 12_000_000 // 4
hx = torch.empty(n, dtype=torch.float32).pin_memory()
hy = torch.empty(n, dtype=torch.float32).pin_memory()
dx = torch.empty(n, dtype=torch.float32, device="cuda")
dy = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ("one", "two", "one", "two"):
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if mode == "one":
            with torch.cuda.stream(s1):
                dx.copy_(hx, non_blocking=True)
                dy.copy_(hy, non_blocking=True)
        else:
            with torch.cuda.stream(s1):
                dx.copy_(hx, non_blocking=True)
            with torch.cuda.stream(s2):
                dy.copy_(hy, non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = sorted(ts)[len(ts) // 2]
    print(f"{mode}: {t*1e3:.3f} ms  {24e6 / t / 1e9:.1f} GB/s")
