"""Calibration only (library kernels, not the product): what do cuDNN / CUTLASS
FMHA kernels reach on this box for the same shapes?"""
import time, sys, math
import torch
import torch.nn.functional as F
from torch.nn.attention import sdpa_kernel, SDPBackend

def bench(fn, iters=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

for (L, h, N, d, dt) in [(4, 16, 4096, 128, torch.float16), (8, 32, 16384, 128, torch.bfloat16), (16, 12, 512, 64, torch.float16), (4, 32, 4096, 64, torch.float16), (2, 8, 8192, 256, torch.float16)]:
    fl = 4 * L * h * N * N * d
    q, k, v = (torch.randn(L, h, N, d, device="cuda", dtype=dt) for _ in range(3))
    for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION):
        try:
            with sdpa_kernel([be]):
                ms = bench(lambda: F.scaled_dot_product_attention(q, k, v))
            print(f"L={L} h={h} N={N} d={d} {dt} {be.name}: {ms:.4f} ms {fl/ms/1e9:.1f} TFLOP/s", flush=True)
        except Exception as ex:
            print(f"L={L} h={h} N={N} d={d} {be.name}: failed {str(ex)[:100]}", flush=True)
    try:
        import flashinfer
        from flashinfer.prefill import fmha_varlen
        qv, kv_, vv = (x.transpose(1, 2).reshape(L * N, h, d).contiguous() for x in (q, k, v))
        off = torch.arange(0, (L + 1) * N, N, device="cuda", dtype=torch.int32)
        t0 = time.time()
        fmha_varlen(qv, kv_, vv, off, off)
        torch.cuda.synchronize()
        ms = bench(lambda: fmha_varlen(qv, kv_, vv, off, off, max_qo_len=N))
        print(f"L={L} h={h} N={N} d={d} {dt} flashinfer-cutlass-sm100: {ms:.4f} ms {fl/ms/1e9:.1f} TFLOP/s (jit {time.time()-t0:.0f}s)", flush=True)
    except Exception as ex:
        print(f"flashinfer cutlass failed: {str(ex)[:300]}", flush=True)
