"""A/B timing of the product kernel on a list of shapes (env selects the variant).
python tools/exp/ab.py TAG  -> one line per shape: TFLOP/s, max |diff| vs the default path's output
saved in /tmp/ab_ref_*.pt by the first (TAG=base) run."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2312_11918_b200 as fm

tag = sys.argv[1]
shapes = [(16, 12, 512, 64, torch.float16), (4, 32, 4096, 64, torch.float16), (4, 16, 4096, 128, torch.float16),
          (8, 32, 16384, 128, torch.bfloat16), (2, 8, 8192, 256, torch.float16), (3, 5, 1000, 64, torch.bfloat16)]
extra = [(4, 16, 4096, 128, torch.bfloat16), (2, 16, 8192, 128, torch.float16), (2, 16, 8192, 128, torch.bfloat16),
         (1, 16, 16384, 128, torch.float16), (8, 16, 2048, 128, torch.float16), (16, 16, 1024, 128, torch.float16),
         (16, 32, 1024, 64, torch.float16), (8, 32, 2048, 64, torch.float16), (2, 32, 8192, 64, torch.float16),
         (4, 32, 4096, 64, torch.bfloat16), (1, 1, 512, 64, torch.float16), (32, 16, 256, 64, torch.float16),
         (16, 12, 768, 64, torch.float16), (4, 16, 4000, 128, torch.float16),
         (1, 20, 1024, 64, torch.bfloat16), (1, 32, 640, 128, torch.float16), (2, 8, 1024, 128, torch.float16),
         (1, 8, 1000, 128, torch.float16)]
shapes += extra
if len(sys.argv) > 2:
    shapes = [shapes[int(i)] for i in sys.argv[2].split(",")]
for (L, h, N, d, dt) in shapes:
    g = torch.Generator(device="cuda").manual_seed(1234)
    q, k, v = (torch.randn(L, N, h, d, device="cuda", dtype=dt, generator=g) for _ in range(3))
    o = fm.fmha_fwd(q, k, v)[0]
    key = f"/tmp/ab_ref_{L}_{h}_{N}_{d}_{str(dt)[6:]}.pt"
    if tag == "base":
        torch.save(o.cpu(), key)
        diff = 0.0
    else:
        diff = (o.float().cpu() - torch.load(key).float()).abs().max().item() if os.path.exists(key) else float("nan")
    iters = max(3, min(50, int(2e13 / (4 * L * h * N * N * d))))
    for _ in range(3):
        fm.fmha_fwd(q, k, v)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for rep in range(3):
        s.record()
        for _ in range(iters):
            fm.fmha_fwd(q, k, v)
        e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / iters)
    fl = 4 * L * h * N * N * d
    print(f"{tag:10s} L={L:2d} h={h:2d} N={N:5d} d={d:3d} {str(dt)[6:]:8s} {best:.4f} ms {fl / best / 1e9:7.1f} TF  maxdiff {diff:.2e}", flush=True)
