import torch, time
n = 200 * 2**20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(68 * 2**20, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(68 * 2**20, dtype=torch.uint8, device="cuda")
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
def t(f, reps=10):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
th = t(lambda: d.copy_(h, non_blocking=True))
td = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
tb = t(both)
print(f"H2D 200MB {th*1e3:.2f} ms = {n/th/1e9:.1f} GB/s; D2H 68MB {td*1e3:.2f} ms = {68*2**20/td/1e9:.1f} GB/s; both concurrently {tb*1e3:.2f} ms")
# chunked H2D
for ch in (4, 16, 64):
    sz = n // ch
    tc_ = t(lambda: [d[i*sz:(i+1)*sz].copy_(h[i*sz:(i+1)*sz], non_blocking=True) for i in range(ch)])
    print(f"H2D in {ch} chunks: {tc_*1e3:.2f} ms")
