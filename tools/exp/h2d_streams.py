"""Pinned H2D rate with 1, 2, 4 concurrent streams (same total bytes), and with a concurrent D2H."""
import torch, time
dev = torch.device("cuda:0")
n = 256 << 20
host = torch.empty(n, dtype=torch.uint8).pin_memory()
dbuf = torch.empty(n, dtype=torch.uint8, device=dev)
host2 = torch.empty(n // 4, dtype=torch.uint8).pin_memory()
dbuf2 = torch.empty(n // 4, dtype=torch.uint8, device=dev)
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream(dev) for _ in range(ns)]
    best = 0
    for rep in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ch = n // ns
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dbuf[i * ch:(i + 1) * ch].copy_(host[i * ch:(i + 1) * ch], non_blocking=True)
        torch.cuda.synchronize()
        best = max(best, n / (time.perf_counter() - t0) / 1e9)
    print(f"H2D {ns} stream(s): {best:.1f} GB/s")
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
best = 0
for rep in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    with torch.cuda.stream(s1): dbuf.copy_(host, non_blocking=True)
    with torch.cuda.stream(s2): host2.copy_(dbuf2, non_blocking=True)
    torch.cuda.synchronize()
    best = max(best, n / (time.perf_counter() - t0) / 1e9)
print(f"H2D with a concurrent D2H of 1/4 the bytes: {best:.1f} GB/s (H2D bytes / wall)")
