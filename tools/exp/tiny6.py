"""d=128 mid-length sequences, many tiles: ping-pong vs single-CTA kBN=64 (two CTAs/SM); cold/large inputs."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2312_11918_b200 as fm
fl = torch.empty(2 * 126 * 2**20 // 4, dtype=torch.float32, device="cuda")
tag = sys.argv[1]
for (L, h, N) in [(8, 16, 1536), (4, 16, 2048), (8, 16, 2048), (4, 16, 3072), (2, 16, 4096), (4, 16, 4096)]:
    q, k, v = (torch.randn(L, N, h, 128, device="cuda").half() for _ in range(3))
    ts = []
    for it in range(15):
        fl.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); o, _ = fm.fmha_fwd(q, k, v); e.record(); torch.cuda.synchronize()
        if it >= 3: ts.append(s.elapsed_time(e))
    ms = sorted(ts)[len(ts) // 2]
    print(f"{tag:5s} L={L:2d} h={h} N={N:5d} tiles={L*h*((N+127)//128):4d} {ms*1e3:7.1f} us {4*L*h*N*N*128/ms/1e9:7.1f} TF {fm.kernel_for(L, N, h, 128)[:24]}", flush=True)
