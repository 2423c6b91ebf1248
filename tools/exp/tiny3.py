"""d=64 one-wave problems: single-CTA kBN=128 (1 CTA/SM) vs kBN=64 (2 CTAs/SM) vs persistent; cold L2, us."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2312_11918_b200 as fm
fl = torch.empty(2 * 126 * 2**20 // 4, dtype=torch.float32, device="cuda")
tag = sys.argv[1]
for (L, h, N) in [(1, 1, 512), (1, 16, 1024), (1, 37, 512), (1, 60, 512), (1, 72, 512), (2, 37, 512), (1, 8, 4096)]:
    q, k, v = (torch.randn(L, N, h, 64, device="cuda").half() for _ in range(3))
    ts = []
    for it in range(25):
        fl.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); o, _ = fm.fmha_fwd(q, k, v); e.record(); torch.cuda.synchronize()
        if it >= 5: ts.append(s.elapsed_time(e))
    ms = sorted(ts)[len(ts) // 2]
    ref = torch.nn.functional.scaled_dot_product_attention(q.transpose(1, 2).float(), k.transpose(1, 2).float(), v.transpose(1, 2).float()).transpose(1, 2)
    err = (o.float() - ref).abs().max().item()
    print(f"{tag:6s} L={L} h={h:2d} N={N:5d} tiles={L*h*((N+127)//128):4d} {ms*1e3:7.1f} us err {err:.1e} {fm.kernel_for(L, N, h, 64)[:24]}", flush=True)
