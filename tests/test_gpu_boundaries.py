"""GPU: every kernel family at and around its dispatch thresholds (DESIGN.md §3,
tests/test_dispatch.py) against a plain PyTorch fp32 attention of the same
16-bit inputs -- O within 2e-2 max abs (bf16) / 5e-3 (fp16) and LSE within
1e-3 relative -- plus the launch count and the kernel the dispatcher names."""
import math

import pytest

pytestmark = pytest.mark.gpu

SHAPES = [  # (L, N, h, d)
    (1, 1024, 37, 64), (1, 1024, 38, 64), (2, 1025, 3, 64),      # one CTA per tile <-> two-CTA d=64
    (3, 8191, 1, 128), (3, 8192, 1, 128), (3, 8193, 1, 128),     # long d=128, ragged last tile
    (1, 512, 37, 64), (1, 512, 38, 64), (1, 4096, 4, 128),       # one CTA per Q tile up to #SMs tiles
    (1, 1000, 40, 64), (3, 2100, 4, 128), (2, 1100, 20, 64),     # ragged N on the persistent kernels
    (2, 333, 40, 64), (1, 512, 38, 64), (2, 700, 21, 128), (1, 300, 99, 64),
    (2, 128, 3, 256), (2, 129, 3, 256), (1, 255, 2, 256), (1, 257, 2, 256),  # single CTA <-> pair d=256
    (3, 640, 5, 128), (4, 96, 7, 64),
    # d=64 below N = 1024: two CTAs per SM once the ping-pong units would fill every SM
    (16, 200, 12, 64), (64, 77, 12, 64), (148, 128, 1, 64), (149, 128, 1, 64), (147, 256, 1, 64),
    (2, 512, 74, 64),
]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("dt", ["f16", "bf16"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "L%d-N%d-h%d-d%d" % s)
def test_kernel_family_boundaries(shape, dt):
    import torch
    import paper_2312_11918_b200 as fm
    L, N, h, d = shape
    td = torch.bfloat16 if dt == "bf16" else torch.float16
    g = torch.Generator(device="cuda").manual_seed(L * 7919 + N * 31 + h * 7 + d)
    q, k, v = (torch.randn((L, N, h, d), generator=g, device="cuda").to(td) for _ in range(3))
    o, lse = fm.fmha_fwd(q, k, v)
    torch.cuda.synchronize()
    assert fm.launch_count() == 1
    name = fm.kernel_for(L, N, h, d, dt)
    tiles = L * h * ((N + 127) // 128)
    if d <= 128 and (tiles <= 148 or (tiles <= 296 and (d == 64 or N <= 2048))):  # one CTA per tile
        assert name.startswith("fmha_fwd_st_kernel"), name
    elif d == 64 and N < 1024:  # the unit-count rule
        assert name.startswith("fmha_fwd_d64_kernel") == (L * h * ((N + 255) // 256) >= 148), name
    qf, kf, vf = (x.float().permute(0, 2, 1, 3) for x in (q, k, v))  # (L, h, N, d)
    s = qf @ kf.transpose(-1, -2) / math.sqrt(d)
    lse_ref = torch.logsumexp(s, dim=-1)                               # (L, h, N)
    o_ref = (torch.softmax(s, dim=-1) @ vf).permute(0, 2, 1, 3)        # (L, N, h, d)
    tol = 2e-2 if dt == "bf16" else 5e-3
    assert float((o.float() - o_ref).abs().max()) < tol
    assert float(((lse - lse_ref).abs() / lse_ref.abs().clamp_min(1.0)).max()) < 1e-3
