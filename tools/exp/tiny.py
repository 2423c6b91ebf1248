"""Tiny problems: cold-L2 time per launch (memset flush) for the default dispatch vs FMHA_TUNE_TINY."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2312_11918_b200 as fm
fl = torch.empty(2 * 126 * 2**20 // 4, dtype=torch.float32, device="cuda")
tag = sys.argv[1]
for (L, h, N, d) in [(1, 1, 512, 64), (1, 1, 256, 64), (1, 2, 512, 64), (1, 1, 1024, 64), (2, 2, 512, 64),
                     (1, 1, 512, 128), (1, 4, 1024, 128), (1, 1, 2048, 128), (4, 8, 512, 64)]:
    q, k, v = (torch.randn(L, N, h, d, device="cuda").half() for _ in range(3))
    ts = []
    for it in range(30):
        fl.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); o, lse = fm.fmha_fwd(q, k, v); e.record(); torch.cuda.synchronize()
        if it >= 5: ts.append(s.elapsed_time(e))
    ms = sorted(ts)[len(ts) // 2]
    ref = torch.nn.functional.scaled_dot_product_attention(q.transpose(1, 2).float(), k.transpose(1, 2).float(), v.transpose(1, 2).float()).transpose(1, 2)
    err = (o.float() - ref).abs().max().item()
    print(f"{tag:5s} L={L} h={h} N={N:5d} d={d:3d} {ms*1e3:7.1f} us {4*L*h*N*N*d/ms/1e9:7.2f} TF err {err:.1e} {fm.kernel_for(L, N, h, d)[:26]}", flush=True)
