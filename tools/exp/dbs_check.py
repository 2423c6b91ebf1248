"""Quick correctness + timing of a d=128 kernel variant (env FMHA_TUNE_* selects it)
against a torch fp32 attention on small shapes; prints the kernel name per shape."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2312_11918_b200 as fm

def ref(q, k, v):
    qf, kf, vf = (x.float().permute(0, 2, 1, 3) for x in (q, k, v))
    s = qf @ kf.transpose(-1, -2) / (q.shape[-1] ** 0.5)
    lse = torch.logsumexp(s, -1)
    o = torch.softmax(s, -1) @ vf
    return o.permute(0, 2, 1, 3), lse

shapes = [(1, 1, 128, 128), (1, 2, 256, 128), (2, 3, 1000, 128), (1, 2, 77, 128), (3, 2, 640, 128),
          (1, 4, 2048, 128), (2, 16, 4096, 128)]
ok = True
for dt in (torch.float16, torch.bfloat16):
    for (L, h, N, d) in shapes:
        g = torch.Generator(device="cuda").manual_seed(N + h)
        q, k, v = (torch.randn(L, N, h, d, device="cuda", generator=g).to(dt) for _ in range(3))
        if N == 640:
            q = q * 4  # force rescales
        o, lse = fm.fmha_fwd(q, k, v)
        torch.cuda.synchronize()
        ro, rl = ref(q, k, v)
        eo = (o.float() - ro).abs()
        el = ((lse - rl).abs() / rl.abs()).max().item()
        tol = 1e-2 if dt == torch.bfloat16 else 4e-3
        good = eo.max().item() <= tol and el <= 1e-4 and torch.isfinite(o).all().item()
        ok &= good
        print(f"{'OK ' if good else 'BAD'} {str(dt)[6:]:8s} L={L} h={h} N={N:5d}: O max {eo.max().item():.2e} mean {eo.mean().item():.2e} LSE rel {el:.2e}  [{fm.kernel_for(L, N, h, d, 1 if dt == torch.bfloat16 else 0)}]", flush=True)
print("ALL OK" if ok else "FAILURES")
