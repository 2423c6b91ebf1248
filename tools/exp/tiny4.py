"""(#SMs, 2 #SMs] Q tiles: persistent kernels vs one CTA per tile with two CTAs per SM; cold L2, us."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2312_11918_b200 as fm
fl = torch.empty(2 * 126 * 2**20 // 4, dtype=torch.float32, device="cuda")
tag = sys.argv[1]
for (L, h, N, d) in [(1, 60, 512, 64), (1, 72, 512, 64), (2, 37, 512, 64), (1, 8, 4096, 64), (1, 19, 1024, 64),
                     (1, 40, 512, 128), (1, 36, 1024, 128), (1, 8, 4096, 128), (1, 4, 8192, 64), (2, 9, 2048, 128)]:
    q, k, v = (torch.randn(L, N, h, d, device="cuda").half() for _ in range(3))
    ts = []
    for it in range(25):
        fl.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); o, _ = fm.fmha_fwd(q, k, v); e.record(); torch.cuda.synchronize()
        if it >= 5: ts.append(s.elapsed_time(e))
    ms = sorted(ts)[len(ts) // 2]
    ref = torch.nn.functional.scaled_dot_product_attention(q.transpose(1, 2).float(), k.transpose(1, 2).float(), v.transpose(1, 2).float()).transpose(1, 2)
    err = (o.float() - ref).abs().max().item()
    print(f"{tag:5s} L={L} h={h:2d} N={N:5d} d={d:3d} tiles={L*h*((N+127)//128):4d} {ms*1e3:7.1f} us err {err:.1e} {fm.kernel_for(L, N, h, d)[:24]}", flush=True)
