"""More than two waves of Q tiles: persistent kernels vs single-CTA kBN=64 (FMHA_TUNE_TINY2 raised); cold L2."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2312_11918_b200 as fm
fl = torch.empty(2 * 126 * 2**20 // 4, dtype=torch.float32, device="cuda")
tag = sys.argv[1]
for (L, h, N, d) in [(4, 16, 1024, 128), (8, 16, 512, 128), (2, 16, 2048, 128), (4, 16, 2048, 128), (16, 16, 512, 128),
                     (4, 24, 512, 64), (8, 16, 1024, 64), (16, 12, 512, 64)]:
    q, k, v = (torch.randn(L, N, h, d, device="cuda").half() for _ in range(3))
    ts = []
    for it in range(25):
        fl.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); o, _ = fm.fmha_fwd(q, k, v); e.record(); torch.cuda.synchronize()
        if it >= 5: ts.append(s.elapsed_time(e))
    ms = sorted(ts)[len(ts) // 2]
    print(f"{tag:5s} L={L:2d} h={h} N={N:5d} d={d:3d} tiles={L*h*((N+127)//128):4d} {ms*1e3:7.1f} us {4*L*h*N*N*d/ms/1e9:7.1f} TF {fm.kernel_for(L, N, h, d)[:24]}", flush=True)
