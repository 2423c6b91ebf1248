"""Randomised shapes through fmha_fwd vs a PyTorch fp32 attention on sampled query rows
(robustness sweep over every kernel family and the dispatch thresholds)."""
import math
import random
import sys

import torch

sys.path.insert(0, ".")
import paper_2312_11918_b200 as fm

random.seed(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
n_cases = int(sys.argv[2]) if len(sys.argv) > 2 else 150
wide = len(sys.argv) > 3 and sys.argv[3] == "wide"  # many heads: the one-/two-CTA-per-tile and wave-quantised paths
worst = {}
for case in range(n_cases):
    d = random.choice([64, 128, 256])
    if wide:
        N = random.choice([random.randint(1, 600), random.randint(600, 4200)])
        L, h = random.randint(1, 4), random.randint(6, 48)
    else:
        N = random.choice([random.randint(1, 300), random.randint(300, 2100), random.randint(7000, 9000)])
        L, h = random.randint(1, 3), random.randint(1, 5)
    dt = random.choice([torch.float16, torch.bfloat16])
    g = torch.Generator(device="cuda").manual_seed(case)
    scale_in = random.choice([0.5, 1.0, 3.0])
    q, k, v = (torch.randn((L, N, h, d), generator=g, device="cuda") * scale_in for _ in range(3))
    q, k, v = (x.to(dt) for x in (q, k, v))
    o, lse = fm.fmha_fwd(q, k, v)
    torch.cuda.synchronize()
    rows = torch.randint(0, N, (min(N, 64),), device="cuda")
    qf = q[:, rows].float().permute(0, 2, 1, 3)                    # L,h,R,d
    kf, vf = (x.float().permute(0, 2, 1, 3) for x in (k, v))        # L,h,N,d
    s = qf @ kf.transpose(-1, -2) / math.sqrt(d)
    o_ref = (torch.softmax(s, -1) @ vf).permute(0, 2, 1, 3)         # L,R,h,d
    lse_ref = torch.logsumexp(s, -1)                               # L,h,R
    err = float((o[:, rows].float() - o_ref).abs().max())
    lerr = float(((lse[:, :, rows] - lse_ref).abs() / lse_ref.abs().clamp_min(1)).max())
    kern = fm.kernel_for(L, N, h, d, "bf16" if dt == torch.bfloat16 else "f16").split(" ")[0]
    tol = (3e-2 if dt == torch.bfloat16 else 8e-3) * max(1.0, scale_in)
    bad = not (err < tol and lerr < 2e-3) or not math.isfinite(err)
    w = worst.setdefault(kern, [0.0, 0.0, 0])
    w[0], w[1], w[2] = max(w[0], err / max(1.0, scale_in)), max(w[1], lerr), w[2] + 1
    if bad:
        print(f"FAIL case {case}: L={L} N={N} h={h} d={d} {dt} x{scale_in} [{kern}] O err {err:.3e} LSE rel {lerr:.3e}")
for kern, (e, l, n) in worst.items():
    print(f"{kern:32s} cases {n:3d}  worst O err / input scale {e:.3e}  worst LSE rel {l:.3e}")
