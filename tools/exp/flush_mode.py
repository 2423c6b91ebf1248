"""c1/c2 device time per launch under two L2-flush methods: a 252 MB memset (dirty lines left in
L2) vs the same memset followed by a read of a second 252 MB buffer (L2 left clean)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2312_11918_b200 as fm
dev = torch.device("cuda:0")
L2 = 126 * 2**20
fl = torch.empty(2 * L2 // 4, dtype=torch.float32, device=dev)
fl2 = torch.ones(2 * L2 // 4, dtype=torch.float32, device=dev)
for (L, h, N, d) in [(16, 12, 512, 64), (1, 1, 512, 64), (4, 16, 4096, 128)]:
    q, k, v = (torch.randn(L, N, h, d, device=dev).half() for _ in range(3))
    for mode in ("memset", "memset+read", "none"):
        ts = []
        for it in range(25):
            if mode != "none":
                fl.zero_()
                if mode == "memset+read":
                    _ = fl2.sum()
            s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
            s.record(); fm.fmha_fwd(q, k, v); e.record(); torch.cuda.synchronize()
            if it >= 5: ts.append(s.elapsed_time(e))
        ms = sum(ts) / len(ts)
        print(f"L={L} h={h} N={N} d={d} {mode:12s} {ms*1e3:7.1f} us  {4*L*h*N*N*d/ms/1e9:7.1f} TF", flush=True)
