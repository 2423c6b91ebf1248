"""d=64 at short N: TFLOP/s for a list of shapes (kernel chosen by FMHA_TUNE_D64_N), cold L2 (memset flush)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2312_11918_b200 as fm
fl = torch.empty(2 * 126 * 2**20 // 4, dtype=torch.float32, device="cuda")
tag = sys.argv[1]
for (L, h, N) in [(16, 12, 128), (16, 12, 200), (16, 12, 256), (16, 12, 384), (16, 12, 512), (16, 12, 640),
                  (16, 12, 768), (16, 12, 1000), (1, 16, 512), (2, 8, 333), (64, 12, 512), (4, 4, 768)]:
    q, k, v = (torch.randn(L, N, h, 64, device="cuda").half() for _ in range(3))
    ts = []
    for it in range(25):
        fl.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fm.fmha_fwd(q, k, v); e.record(); torch.cuda.synchronize()
        if it >= 5: ts.append(s.elapsed_time(e))
    ms = sorted(ts)[len(ts) // 2]
    print(f"{tag:6s} L={L:2d} h={h:2d} N={N:5d} {ms*1e3:8.1f} us {4*L*h*N*N*64/ms/1e9:7.1f} TF  {fm.kernel_for(L, N, h, 64)[:22]}", flush=True)
