"""Host-only: which kernel the dispatcher picks (fmha_kernel_for, no CUDA call).
The thresholds are the measured crossovers documented in DESIGN.md §3."""
import pytest

import paper_2312_11918_b200 as fm


@pytest.mark.parametrize("shape,kernel", [
    ((1, 512, 1, 64), "fmha_fwd_st_kernel<64|128,128>"),  # c1: 4 Q tiles, one CTA each
    ((1, 4096, 4, 128), "fmha_fwd_st_kernel<64|128,128>"),  # 128 Q tiles <= 148 SMs
    ((1, 512, 37, 64), "fmha_fwd_st_kernel<64|128,128>"),  # 148 Q tiles
    ((1, 512, 38, 64), "fmha_fwd_st_kernel<64|128,64>"),   # 152 Q tiles: one CTA per tile, two per SM
    ((1, 1024, 37, 64), "fmha_fwd_st_kernel<64|128,64>"),  # 296 Q tiles
    ((1, 1024, 38, 64), "fmha_fwd_d64_kernel"),           # 304 Q tiles, N >= 1024
    ((1, 512, 75, 64), "fmha_fwd_d64_kernel"),            # 300 Q tiles, 150 ping-pong units
    ((16, 512, 12, 64), "fmha_fwd_d64_kernel"),           # c2: 768 Q tiles
    ((4, 4096, 32, 64), "fmha_fwd_d64_kernel"),           # Table-1 d=64
    ((1, 2048, 18, 128), "fmha_fwd_st_kernel<64|128,64>"),  # 288 Q tiles, N <= 2048
    ((1, 4096, 8, 128), "fmha_fwd_sm100_kernel<128>"),    # 256 Q tiles but N > 2048
    ((4, 4096, 16, 128), "fmha_fwd_sm100_kernel<128>"),   # c3: 1024 units, wave efficiency 0.99
    ((2, 4096, 16, 128), "fmha_fwd_sm100_kernel<128>"),   # 512 units (wave efficiency 0.86: still persistent)
    ((8, 2048, 16, 128), "fmha_fwd_sm100_kernel<128>"),   # 1024 units
    ((16, 1024, 16, 128), "fmha_fwd_sm100_kernel<128>"),
    ((3, 8192, 1, 128), "fmha_fwd_sm100_kernel<128>"),    # long d=128: ping-pong (CTA pairs are opt-in)
    ((8, 16384, 32, 128), "fmha_fwd_sm100_kernel<128>"),  # c5
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


@pytest.mark.parametrize("env,shape,kernel", [
    ({"FMHA_TUNE_PAIR128_N": "8192"}, (1, 8192, 3, 128), "fmha_fwd_pair_kernel<128,64>"),  # opt-in d=128 pairs
    ({"FMHA_TUNE_PAIR128_N": "8192"}, (1, 4096, 8, 128), "fmha_fwd_sm100_kernel<128>"),    # below the cut
    ({"FMHA_TUNE_PAIR": "0"}, (2, 8192, 8, 256), "fmha_fwd_st_kernel<256,128>"),          # no CTA pairs at all
    ({"FMHA_TUNE_DBS": "1"}, (4, 4096, 16, 128), "fmha_fwd_dbs_kernel<128>"),
    ({"FMHA_TUNE_TINY": "0", "FMHA_TUNE_TINY2": "0"}, (1, 512, 1, 64), "fmha_fwd_sm100_kernel<64>"),
    ({"FMHA_TUNE_D64": "0"}, (16, 512, 12, 64), "fmha_fwd_sm100_kernel<64>"),
])
def test_kernel_choice_overrides(env, shape, kernel):
    """The FMHA_TUNE_* overrides (read once per process, so each case runs in a
    subprocess; host-only, no CUDA call)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = f"import paper_2312_11918_b200 as fm; print(fm.kernel_for(*{shape!r}))"
    out = subprocess.run([sys.executable, "-c", code], check=True, cwd=root, capture_output=True, text=True,
                         env=dict(os.environ, **env), timeout=120).stdout
    assert out.startswith(kernel), out
