"""Host-only: which kernel the dispatcher picks (fmha_kernel_for, no CUDA call).
The thresholds are the measured crossovers documented in DESIGN.md §3."""
import pytest

import paper_2312_11918_b200 as fm


@pytest.mark.parametrize("shape,kernel", [
    ((1, 512, 1, 64), "fmha_fwd_sm100_kernel<64>"),       # c1
    ((16, 512, 12, 64), "fmha_fwd_d64_kernel"),           # c2: 384 ping-pong units fill every SM
    ((1, 512, 16, 64), "fmha_fwd_sm100_kernel<64>"),      # few heads, short N
    ((4, 768, 4, 64), "fmha_fwd_sm100_kernel<64>"),
    ((4, 1024, 32, 64), "fmha_fwd_d64_kernel"),           # d=64 from N = 1024
    ((4, 4096, 32, 64), "fmha_fwd_d64_kernel"),           # Table-1 d=64
    ((4, 4096, 16, 128), "fmha_fwd_sm100_kernel<128>"),   # c3
    ((1, 8191, 2, 128), "fmha_fwd_sm100_kernel<128>"),
    ((1, 8192, 2, 128), "fmha_fwd_pair_kernel<128,64>"),
    ((8, 16384, 32, 128), "fmha_fwd_pair_kernel<128,64>"),  # c5
    ((2, 8192, 8, 256), "fmha_fwd_pair_kernel<256,128>"),  # c4
    ((1, 129, 2, 256), "fmha_fwd_pair_kernel<256,128>"),   # two Q tiles (one padded)
    ((1, 128, 2, 256), "fmha_fwd_st_kernel<256,128>"),     # a single Q tile
])
def test_kernel_choice(shape, kernel):
    assert fm.kernel_for(*shape).startswith(kernel)


def test_kernel_choice_rejects_invalid_problems():
    with pytest.raises(ValueError):
        fm.kernel_for(1, 0, 1, 64)
    with pytest.raises(ValueError):
        fm.kernel_for(1, 128, 1, 96)  # head dim without a kernel
