"""Run-to-run determinism of the product path: the same inputs N times, bitwise comparison."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2312_11918_b200 as fm
for (L, h, N, d, dt) in [(4, 16, 4096, 128, torch.float16), (4, 16, 4096, 128, torch.bfloat16), (16, 12, 512, 64, torch.float16),
                         (8, 16, 2048, 128, torch.float16), (2, 8, 8192, 256, torch.float16)]:
    g = torch.Generator(device="cuda").manual_seed(1234)
    q, k, v = (torch.randn(L, N, h, d, device="cuda", dtype=dt, generator=g) for _ in range(3))
    o0, l0 = fm.fmha_fwd(q, k, v)
    o0 = o0.clone(); l0 = l0.clone()
    bad = 0; worst = 0.0
    for r in range(20):
        o, l = fm.fmha_fwd(q, k, v)
        if not (torch.equal(o, o0) and torch.equal(l, l0)):
            bad += 1
            worst = max(worst, (o.float() - o0.float()).abs().max().item())
    torch.cuda.synchronize()
    print(f"L={L} h={h} N={N} d={d} {str(dt)[6:]}: {bad}/20 runs differ from the first (max |dO| {worst:.2e}) [{fm.kernel_for(L, N, h, d, 1 if dt == torch.bfloat16 else 0)}]", flush=True)
