"""Small ragged/bf16/d=256 cases for compute-sanitizer runs:
    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_smoke.py
Results and their reading: DESIGN.md §10."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2312_11918_b200 as fm
torch.manual_seed(0)
only_d128 = len(sys.argv) > 1 and sys.argv[1] == "d128"  # (with FMHA_TUNE_DBS=1: the double-buffered-S kernel)
pair128 = len(sys.argv) > 1 and sys.argv[1] == "pair128"  # (with FMHA_TUNE_PAIR128_N=8192: the d=128 CTA-pair kernel)
cases = [(1, 8320, 3, 128, torch.bfloat16), (2, 8192, 2, 128, torch.float16)] if pair128 else [(1, 77, 2, 128, torch.float16), (2, 333, 3, 128, torch.bfloat16), (3, 130, 1, 128, torch.float16),
         (1, 1000, 150, 128, torch.float16)] if only_d128 else [(1, 200, 2, 64, torch.float16), (2, 333, 3, 128, torch.bfloat16), (1, 1000, 2, 256, torch.float16), (3, 130, 1, 128, torch.float16), (1, 1, 1, 64, torch.float16),
                         (1, 1100, 2, 64, torch.float16),      # d=64 two-CTA-per-SM kernel
                         (16, 200, 12, 64, torch.bfloat16),    # the same below N = 1024 (many heads)
                         (1, 384, 2, 256, torch.bfloat16),     # CTA pair with a padding tile
                         (1, 8320, 1, 128, torch.bfloat16)]    # long d=128, one CTA per Q tile
for (L, N, h, d, dt) in cases:
    if pair128:
        assert "pair_kernel<128,64>" in fm.kernel_for(L, N, h, d, fm.BF16 if dt == torch.bfloat16 else fm.F16)
    q, k, v = (torch.randn(L, N, h, d, device="cuda", dtype=dt) for _ in range(3))
    o, lse = fm.fmha_fwd(q, k, v)
    torch.cuda.synchronize()
    ref = torch.nn.functional.scaled_dot_product_attention(q.transpose(1, 2).float(), k.transpose(1, 2).float(), v.transpose(1, 2).float()).transpose(1, 2)
    err = (o.float() - ref).abs().max().item()
    print(L, N, h, d, dt, "max err", err, flush=True)
    assert err < 3e-2, "output mismatch"
