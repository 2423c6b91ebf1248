"""Per-call latency of small problems through fmha_fwd (host descriptor encode +
launch + kernel), CUDA-event timed back-to-back calls and host wall time per call."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2312_11918_b200 as fm
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for (L, h, N, d) in [(1, 1, 512, 64), (1, 1, 128, 128), (2, 4, 256, 256), (16, 12, 512, 64)]:
    q, k, v = (torch.randn(L, N, h, d, device="cuda").half() for _ in range(3))
    o = torch.empty_like(q); lse = torch.empty(L, h, N, device="cuda")
    for _ in range(10): fm.fmha_fwd(q, k, v, o=o, lse=lse)
    torch.cuda.synchronize()
    n = 200
    t = time.perf_counter()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fm.fmha_fwd(q, k, v, o=o, lse=lse)
    b.record(); torch.cuda.synchronize()
    wall = (time.perf_counter() - t) / n * 1e6
    print(f"{tag:6s} L={L} h={h} N={N} d={d}: {a.elapsed_time(b) / n * 1e3:.1f} us/call (device), {wall:.1f} us/call (host)")
