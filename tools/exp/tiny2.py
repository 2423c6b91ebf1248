"""Crossover of the one-CTA-per-Q-tile path: cold-L2 us per launch, default vs FMHA_TUNE_TINY=100000."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2312_11918_b200 as fm
fl = torch.empty(2 * 126 * 2**20 // 4, dtype=torch.float32, device="cuda")
tag = sys.argv[1]
for (L, h, N, d) in [(1, 8, 1024, 64), (1, 16, 1024, 64), (1, 36, 512, 64), (1, 37, 512, 64), (1, 72, 512, 64),
                     (1, 8, 1024, 128), (1, 16, 1024, 128), (1, 18, 1024, 128), (1, 36, 1024, 128), (1, 8, 2048, 128),
                     (1, 4, 4096, 128), (1, 9, 2048, 128)]:
    q, k, v = (torch.randn(L, N, h, d, device="cuda").half() for _ in range(3))
    ts = []
    for it in range(25):
        fl.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fm.fmha_fwd(q, k, v); e.record(); torch.cuda.synchronize()
        if it >= 5: ts.append(s.elapsed_time(e))
    ms = sorted(ts)[len(ts) // 2]
    tiles = L * h * ((N + 127) // 128)
    print(f"{tag:5s} L={L} h={h:2d} N={N:5d} d={d:3d} tiles={tiles:4d} {ms*1e3:7.1f} us {4*L*h*N*N*d/ms/1e9:7.1f} TF {fm.kernel_for(L, N, h, d)[:22]}", flush=True)
