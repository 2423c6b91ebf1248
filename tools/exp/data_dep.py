"""Does the d=128 kernel's speed depend on the input data?  c3 shape, Q scaled by s."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2312_11918_b200 as fm
L, h, N, d = 4, 16, 4096, 128
for s in [1.0, 0.1, 0.0, 3.0]:
    g = torch.Generator(device="cuda").manual_seed(1)
    q, k, v = (torch.randn(L, N, h, d, device="cuda", generator=g).half() for _ in range(3))
    q = (q.float() * s).half()
    for _ in range(3): fm.fmha_fwd(q, k, v)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(30): fm.fmha_fwd(q, k, v)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 30
    print(f"q scale {s}: {ms:.4f} ms {4*L*h*N*N*d/ms/1e9:.1f} TF", flush=True)
