"""GPU parity: the sm_100a kernel vs the CPU oracle on identical inputs.

Every test calls through the C ABI (fmha_fwd via ctypes).  Inputs are the
reference's seeded Gaussians (random.hpp:44-50, seeds 42/43/44 as
fmha_cli.cpp:79-84) pre-rounded to the 16-bit type, so the GPU and the
oracle see bit-identical values.
"""
import numpy as np
import pytest

from parity import assert_within, errors, gpu_fmha

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2312_11918_b200 as fm
    fm.lib()


def _full_check(oracle, L, N, h, d, dt, seed=42, scale=None):
    q, k, v = oracle.problem(L, N, h, d, seed, dtype=dt)
    o, lse = gpu_fmha(q, k, v, dt, scale=scale)
    bm = 128 if N % 128 == 0 else N
    o_ref, lse_ref = oracle.fmha_forward(q, k, v, bm, bm, scale=scale)
    res = errors(o, lse, o_ref, lse_ref)
    assert_within(res, f"L={L} N={N} h={h} d={d} {dt}")
    return res


@pytest.mark.parametrize("dt", ["f16", "bf16"])
def test_config1_against_reference_fixture(oracle, dt):
    """c1 (L=1,h=1,N=512,d=64) against outputs of the REFERENCE itself
    (tests/golden/c1_ref.npz, made by tests/golden/make_goldens.py)."""
    import os
    fx = np.load(os.path.join(os.path.dirname(__file__), "golden", "c1_ref.npz"))
    q, k, v = oracle.problem(1, 512, 1, 64, 42, dtype=dt)
    o, lse = gpu_fmha(q, k, v, dt)
    res = errors(o.reshape(512, 64), lse.reshape(512), fx[f"O_{dt}"], fx[f"lse_{dt}"])
    assert_within(res, f"c1 {dt}")


@pytest.mark.parametrize("d", [64, 128, 256])
@pytest.mark.parametrize("dt", ["f16", "bf16"])
def test_small_full(oracle, d, dt):
    _full_check(oracle, 2, 512, 3, d, dt, seed=7)


@pytest.mark.parametrize("N", [1024, 2048])
@pytest.mark.parametrize("dt", ["f16", "bf16"])
def test_d64_two_ctas_per_sm_full(oracle, N, dt):
    """d = 64, more than 2 x #SMs Q tiles: the two-CTA-per-SM kernel (64-row K/V steps)."""
    import paper_2312_11918_b200 as fm
    assert fm.kernel_for(1, N, 40, 64).startswith("fmha_fwd_d64_kernel")
    _full_check(oracle, 1, N, 40, 64, dt, seed=13)


@pytest.mark.parametrize("shape", [(2, 512, 3, 64), (2, 512, 3, 128), (1, 1000, 2, 64), (1, 1000, 2, 128),
                                   (1, 1024, 3, 64), (3, 640, 5, 128)])
def test_persistent_kernels_small_shapes(oracle, tmp_path, shape):
    """Small problems run one CTA per Q tile by default; with that path switched
    off (FMHA_TUNE_TINY=0, FMHA_TUNE_TINY2=0, read once per process: a
    subprocess) they exercise the persistent ping-pong / two-CTA kernels,
    including ragged N, against the oracle."""
    import os
    import subprocess
    import sys
    L, N, h, d = shape
    q, k, v = oracle.problem(L, N, h, d, 77, dtype="f16")
    np.savez(tmp_path / "in.npz", q=q, k=k, v=v)
    code = ("import numpy as np, torch, paper_2312_11918_b200 as fm\n"
            f"z = np.load({str(tmp_path / 'in.npz')!r})\n"
            "q, k, v = (torch.from_numpy(z[x]).cuda().half() for x in ('q', 'k', 'v'))\n"
            f"assert not fm.kernel_for({L}, {N}, {h}, {d}).startswith('fmha_fwd_st_kernel')\n"
            "o, lse = fm.fmha_fwd(q, k, v)\n"
            f"np.savez({str(tmp_path / 'out.npz')!r}, o=o.float().cpu().numpy(), lse=lse.cpu().numpy())\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, "-c", code], check=True, cwd=root, timeout=300,
                   env=dict(os.environ, FMHA_TUNE_TINY="0", FMHA_TUNE_TINY2="0"))
    out = np.load(tmp_path / "out.npz")
    bm = 128 if N % 128 == 0 else N
    o_ref, lse_ref = oracle.fmha_forward(q, k, v, bm, bm)
    assert_within(errors(out["o"], out["lse"], o_ref, lse_ref), f"persistent L={L} N={N} h={h} d={d}")


def test_config2_distilbert_full(oracle):
    """c2: L=16, h=12, N=512, d=64 fp16 -- full O and LSE."""
    _full_check(oracle, 16, 512, 12, 64, "f16")


@pytest.mark.parametrize("N", [1, 37, 128, 200, 384, 640, 1000, 1100])
@pytest.mark.parametrize("d", [64, 128, 256])
def test_ragged_sequence_lengths(oracle, N, d):
    """N not a multiple of the kernel tiles: padded K/V columns are masked,
    padded Q rows are not stored."""
    q, k, v = oracle.problem(1, N, 2, d, 100 + N, dtype="f16")
    o, lse = gpu_fmha(q, k, v, "f16")
    o_ref, lse_ref = oracle.fmha_forward(q, k, v, N, N)  # one tile = standard attention
    assert_within(errors(o, lse, o_ref, lse_ref), f"N={N} d={d}")


def test_single_key_returns_value(oracle):
    """N = 1: the softmax of a single score is 1, so O == V (test_attention.cpp:69-77)."""
    q, k, v = oracle.problem(2, 1, 4, 128, 5, dtype="f16")
    o, lse = gpu_fmha(q, k, v, "f16")
    np.testing.assert_array_equal(o, v)


def test_identical_keys_give_column_mean(oracle):
    """Identical K rows: P uniform, O = column mean of V (test_attention.cpp:79-94)."""
    L, N, h, d = 1, 512, 2, 64
    q, _, v = oracle.problem(L, N, h, d, 3, dtype="f16")
    k = np.zeros_like(q)
    k[...] = (np.arange(d, dtype=np.float32) * 0.25)[None, None, None, :]
    k = oracle.quantize(k, "f16")
    o, lse = gpu_fmha(q, k, v, "f16")
    mean = v.astype(np.float64).mean(axis=1, keepdims=True)
    assert np.abs(o - mean).max() < 2e-3
    # every score in a row equals q.k0 * scale, so LSE = q.k0 * scale + ln N
    s = (q.astype(np.float64) @ k[0, 0, 0].astype(np.float64))[..., None] / np.sqrt(d)
    expect = np.transpose(s[..., 0], (0, 2, 1)) + np.log(N)
    np.testing.assert_allclose(lse, expect, rtol=1e-5, atol=1e-5)


def test_custom_scale(oracle):
    _full_check(oracle, 1, 256, 2, 128, "f16", scale=0.05)


@pytest.mark.parametrize("d,N", [(128, 384), (256, 512), (64, 1024)], ids=["d128", "d256-pair", "d64-two-ctas"])
def test_strided_views(oracle, d, N):
    """Q/K/V as views into one packed (L, N, 3, h, d) buffer and O into a
    padded buffer: the ABI's explicit strides (head-sharding path, 8(e)).
    d = 256 with an even Q-tile count runs the CTA-pair kernel (its K map has
    64-row boxes over the same strides)."""
    import torch
    import paper_2312_11918_b200 as fm
    L, h = 2, 3
    q, k, v = oracle.problem(L, N, h, d, 11, dtype="bf16")
    packed = torch.from_numpy(np.stack([q, k, v], axis=2)).cuda().to(torch.bfloat16)
    out = torch.zeros((L, N, h + 1, d), dtype=torch.bfloat16, device="cuda")
    o_view = out[:, :, 1:, :]
    fm.fmha_fwd(packed[:, :, 0], packed[:, :, 1], packed[:, :, 2], o=o_view)
    torch.cuda.synchronize()
    o_ref, lse_ref = oracle.fmha_forward(q, k, v, 128, 128)
    res = errors(o_view.float().cpu().numpy(), None, o_ref, None)
    assert_within(res, "strided")
    assert float(out[:, :, 0].abs().max()) == 0.0


@pytest.mark.parametrize("cfg", [(4, 4096, 16, 128, "f16"), (2, 8192, 8, 256, "f16"),
                                 (8, 16384, 32, 128, "bf16"), (1, 8320, 2, 128, "f16"),
                                 (1, 2432, 3, 256, "bf16"), (4, 4096, 32, 64, "f16")],
                         ids=["c3", "c4", "c5", "d128-long-odd-tiles", "d256-pair-odd-tiles", "table1-d64"])
def test_large_configs_sampled(oracle, cfg):
    """c3/c4/c5 at full size: inputs generated on the device (seeded torch
    RNG, rounded to the 16-bit type), every (b, head) computed on the GPU,
    and a sample of Q tiles -- first, last and a random one, for the first and
    last head of every batch -- checked against the oracle on the host."""
    import torch
    import paper_2312_11918_b200 as fm
    L, N, h, d, dt = cfg
    td = torch.bfloat16 if dt == "bf16" else torch.float16
    g = torch.Generator(device="cuda").manual_seed(1234)
    q, k, v = (torch.randn((L, N, h, d), generator=g, device="cuda", dtype=torch.float32).to(td) for _ in range(3))
    o, lse = fm.fmha_fwd(q, k, v)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    n_tiles = N // 128
    heads = sorted({(b, hh) for b in range(L) for hh in (0, h - 1)})
    if L > 2:
        heads = [x for x in heads if x[0] in (0, L // 2, L - 1)]
    for (b, hh) in heads:
        qh, kh, vh = (t[b:b + 1, :, hh:hh + 1, :].float().cpu().numpy() for t in (q, k, v))
        tiles = sorted({0, n_tiles - 1, int(rng.integers(n_tiles))})
        o_ref, lse_ref = oracle.fmha_tiles(qh, kh, vh, [(0, 0, i) for i in tiles], 128, 128)
        o_got = np.stack([o[b, i * 128:(i + 1) * 128, hh].float().cpu().numpy() for i in tiles])
        lse_got = np.stack([lse[b, hh, i * 128:(i + 1) * 128].cpu().numpy() for i in tiles])
        assert_within(errors(o_got, lse_got, o_ref, lse_ref), f"{cfg} b={b} h={hh} tiles={tiles}")
    # size-independent properties over the whole output
    assert torch.isfinite(o.float()).all()
    assert torch.isfinite(lse).all()
    # O rows are convex combinations of V rows: within [min V, max V] per column
    vmin = v.float().amin(dim=1, keepdim=True)
    vmax = v.float().amax(dim=1, keepdim=True)
    of = o.float()
    assert bool(((of >= vmin - 2e-2) & (of <= vmax + 2e-2)).all())


def test_kv_permutation_invariance(oracle):
    """Jointly permuting K/V rows changes O only by reassociation
    (test_attention.cpp:262-279), at a multi-tile size."""
    import torch
    import paper_2312_11918_b200 as fm
    L, N, h, d = 1, 2048, 4, 128
    q, k, v = oracle.problem(L, N, h, d, 77, dtype="f16")
    tq, tk, tv = (torch.from_numpy(x).cuda().half() for x in (q, k, v))
    o1, l1 = fm.fmha_fwd(tq, tk, tv)
    perm = torch.randperm(N, generator=torch.Generator().manual_seed(3)).cuda()
    o2, l2 = fm.fmha_fwd(tq, tk[:, perm].contiguous(), tv[:, perm].contiguous())
    torch.cuda.synchronize()
    assert float((o1.float() - o2.float()).abs().max()) < 2e-3
    assert float(((l1 - l2).abs() / l1.abs()).max()) < 1e-5


def test_linearity_in_v(oracle):
    """O is linear in V for fixed Q, K (P does not depend on V)."""
    import torch
    import paper_2312_11918_b200 as fm
    L, N, h, d = 1, 1024, 2, 64
    q, k, v = oracle.problem(L, N, h, d, 21, dtype="f16")
    tq, tk, tv = (torch.from_numpy(x).cuda().half() for x in (q, k, v))
    o1, _ = fm.fmha_fwd(tq, tk, tv)
    o2, _ = fm.fmha_fwd(tq, tk, (tv.float() * 0.5).half())
    torch.cuda.synchronize()
    assert float((o1.float() * 0.5 - o2.float()).abs().max()) < 1e-3


def test_host_entry_points(oracle):
    """fmha_forward (reference call shape, float32 host arrays) and
    fmha_fwd_host (16-bit host buffers) -- copies inside the call."""
    import paper_2312_11918_b200 as fm
    q, k, v = oracle.problem(2, 256, 2, 64, 9)
    o, lse = fm.fmha_forward(q, k, v, 64, 64, precision="f16emu", return_lse=True)
    qq, kk, vv = (oracle.quantize(x, "f16") for x in (q, k, v))
    o_ref, lse_ref = oracle.fmha_forward(qq, kk, vv, 128, 128)
    assert_within(errors(o, lse, o_ref, lse_ref), "fmha_forward host")
    bits = [oracle.to_bits(x, "f16") for x in (qq, kk, vv)]
    o16 = np.empty_like(bits[0])
    lse2 = np.empty((2, 2, 256), np.float32)
    fm.fmha_fwd_host(*bits, o16, lse2, dtype=fm.F16)
    assert_within(errors(oracle.from_bits(o16, "f16"), lse2, o_ref, lse_ref), "fmha_fwd_host")
    with pytest.raises(ValueError):
        fm.fmha_forward(q[:, :100], k[:, :100], v[:, :100], 64, 64)


def test_launch_count():
    import torch
    import paper_2312_11918_b200 as fm
    q = torch.randn(1, 256, 1, 64, device="cuda").half()
    fm.fmha_fwd(q, q, q)
    assert fm.launch_count() == 1


@pytest.mark.parametrize("L,N,h,d,dt", [
    (2, 4096, 16, 128, "f16"),   # 1 batch per input chunk, O/LSE returned in 4 head groups (2-D copies)
    (8, 512, 8, 64, "bf16"),     # several batches per input chunk
    (3, 2048, 6, 256, "f16"),    # d=256 kernel behind the pipeline
    (2, 2048, 4, 64, "f16"),     # last batch split into query-row slices (d=64 kernel)
    (1, 1100, 3, 128, "bf16"),   # row slices with a ragged last slice
])
def test_host_pipeline_bitwise_equals_device_path(L, N, h, d, dt):
    """fmha_fwd_host splits the problem into (batch, head-group) chunks over
    three streams, and the last batch of a long sequence into query-row
    slices; every chunk is an independent sub-problem, so the result must
    equal the single-launch device path bit for bit."""
    import torch
    import paper_2312_11918_b200 as fm
    td = torch.bfloat16 if dt == "bf16" else torch.float16
    g = torch.Generator(device="cuda").manual_seed(11)
    q, k, v = (torch.randn((L, N, h, d), generator=g, device="cuda").to(td) for _ in range(3))
    o_dev, lse_dev = fm.fmha_fwd(q, k, v)
    torch.cuda.synchronize()
    hq, hk, hv = (x.cpu().view(torch.int16).numpy() for x in (q, k, v))
    ho = np.empty_like(hq)
    hl = np.empty((L, h, N), np.float32)
    fm.fmha_fwd_host(hq, hk, hv, ho, hl, dtype=fm.BF16 if dt == "bf16" else fm.F16)
    assert fm.launch_count() >= 1
    assert np.array_equal(ho, o_dev.cpu().view(torch.int16).numpy())
    assert np.array_equal(hl, lse_dev.cpu().numpy())


def test_pair_kernel_matches_single_cta_kernel_bitwise(oracle, tmp_path):
    """d = 256: the CTA-pair kernel (cta_group::2, M = 256) and the single-CTA
    kernel issue the same MMA K-order and the same softmax, so O and LSE are
    bitwise equal.  The single-CTA path is forced in a subprocess
    (FMHA_TUNE_PAIR=0 is read once per process)."""
    import os
    import subprocess
    import sys
    import torch
    import paper_2312_11918_b200 as fm
    L, N, h, d = 1, 1152, 2, 256   # 9 Q tiles: the pair path pads the last unit
    q, k, v = oracle.problem(L, N, h, d, 31, dtype="f16")
    np.savez(tmp_path / "in.npz", q=q, k=k, v=v)
    tq, tk, tv = (torch.from_numpy(x).cuda().half() for x in (q, k, v))
    o, lse = fm.fmha_fwd(tq, tk, tv)
    torch.cuda.synchronize()
    code = (
        "import numpy as np, torch, paper_2312_11918_b200 as fm\n"
        f"z = np.load({str(tmp_path / 'in.npz')!r})\n"
        "q, k, v = (torch.from_numpy(z[n]).cuda().half() for n in ('q', 'k', 'v'))\n"
        "o, lse = fm.fmha_fwd(q, k, v)\n"
        f"np.savez({str(tmp_path / 'out.npz')!r}, o=o.float().cpu().numpy(), lse=lse.cpu().numpy())\n")
    env = dict(os.environ, FMHA_TUNE_PAIR="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, "-c", code], check=True, env=env, cwd=root, timeout=300)
    ref = np.load(tmp_path / "out.npz")
    np.testing.assert_array_equal(o.float().cpu().numpy(), ref["o"])
    np.testing.assert_array_equal(lse.cpu().numpy(), ref["lse"])


@pytest.mark.parametrize("dt", ["f16", "bf16"])
def test_opt_in_d128_pair_kernel_against_oracle(oracle, tmp_path, dt):
    """The d = 128 CTA-pair kernel (cta_group::2, one Q tile per CTA, two CTAs
    per SM) is opt-in since the ping-pong kernel overtook it at long N
    (FMHA_TUNE_PAIR128_N=8192, read once per process: a subprocess).  N = 8320
    (an odd Q-tile count per head: each head's last pair has a padding CTA) plus an even case,
    sampled Q tiles against the tile oracle."""
    import os
    import subprocess
    import sys
    cases = [(1, 8320, 3), (1, 8192, 3)]  # > #SMs Q tiles: past the one-CTA-per-tile paths
    probs = {}
    for n, (L, N, h) in enumerate(cases):
        q, k, v = oracle.problem(L, N, h, 128, 70 + n, dtype=dt)
        probs[n] = (q, k, v)
        np.savez(tmp_path / f"in{n}.npz", q=q, k=k, v=v)
    code = (
        "import numpy as np, torch, paper_2312_11918_b200 as fm\n"
        f"td = torch.bfloat16 if {dt!r} == 'bf16' else torch.float16\n"
        f"for n in range({len(cases)}):\n"
        f"    z = np.load({str(tmp_path)!r} + f'/in{{n}}.npz')\n"
        "    q, k, v = (torch.from_numpy(z[x]).cuda().to(td) for x in ('q', 'k', 'v'))\n"
        "    L, N, h, d = q.shape\n"
        "    assert 'pair_kernel<128,64>' in fm.kernel_for(L, N, h, d, fm.BF16 if td == torch.bfloat16 else fm.F16)\n"
        "    o, lse = fm.fmha_fwd(q, k, v)\n"
        f"    np.savez({str(tmp_path)!r} + f'/out{{n}}.npz', o=o.float().cpu().numpy(), lse=lse.cpu().numpy())\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, "-c", code], check=True, env=dict(os.environ, FMHA_TUNE_PAIR128_N="8192"),
                   cwd=root, timeout=600)
    for n, (L, N, h) in enumerate(cases):
        q, k, v = probs[n]
        out = np.load(tmp_path / f"out{n}.npz")
        tiles = [(0, hh, t) for hh in (0, h - 1) for t in (0, 31, (N - 1) // 128)]
        o_ref, lse_ref = oracle.fmha_tiles(q, k, v, tiles, 128, 128)
        for ti, (b, hh, t) in enumerate(tiles):
            r0, r1 = t * 128, min(N, t * 128 + 128)
            res = errors(out["o"][b, r0:r1, hh], out["lse"][b, hh, r0:r1], o_ref[ti][: r1 - r0],
                         lse_ref[ti][: r1 - r0])
            assert_within(res, f"pair128 {dt} N={N} h={h} tile {(b, hh, t)}")


@pytest.mark.parametrize("env", ["FMHA_TUNE_DBS", "FMHA_TUNE_SPLIT"])
@pytest.mark.parametrize("dt", ["f16", "bf16"])
def test_opt_in_d128_kernels_against_oracle(oracle, tmp_path, dt, env):
    """The opt-in d = 128 kernels -- double-buffered S (FMHA_TUNE_DBS=1) and the
    split-row ping-pong (FMHA_TUNE_SPLIT=1); read once per process, so they
    run in a subprocess -- against the oracle: ragged N
    (masked last K/V step, TMA-clipped Q rows), several units per CTA (the
    flat step sequence crosses unit boundaries with an odd step count), and
    keys growing along the sequence, which force conditional O rescales in
    the speculative half."""
    import os
    import subprocess
    import sys
    # (bf16 takes a milder key ramp: with 3x, P's 8-bit mantissa alone puts both
    # d = 128 kernels at ~1.2e-2, tools/exp/dbs_bf16.py)
    ramp_top = 3.0 if dt == "f16" else 2.0
    cases = [(1, 77, 2, 1.0), (2, 1000, 3, 1.0), (1, 640, 2, ramp_top), (2, 384, 150, 1.0)]
    probs = {}
    for n, (L, N, h, s) in enumerate(cases):
        q, k, v = oracle.problem(L, N, h, 128, 50 + n, dtype=dt)
        if s != 1.0:  # keys growing along the sequence: row maxima keep rising -> O rescales
            ramp = (1.0 + (s - 1.0) * np.arange(N, dtype=np.float32) / N)[None, :, None, None]
            k = oracle.quantize((k * ramp).astype(np.float32), dt)
        probs[n] = (q, k, v)
        np.savez(tmp_path / f"in{n}.npz", q=q, k=k, v=v)
    code = (
        "import numpy as np, torch, paper_2312_11918_b200 as fm\n"
        f"td = torch.bfloat16 if {dt!r} == 'bf16' else torch.float16\n"
        f"for n in range({len(cases)}):\n"
        f"    z = np.load({str(tmp_path)!r} + f'/in{{n}}.npz')\n"
        "    q, k, v = (torch.from_numpy(z[x]).cuda().to(td) for x in ('q', 'k', 'v'))\n"
        "    L, N, h, d = q.shape[0], q.shape[1], q.shape[2], q.shape[3]\n"
        f"    assert {env!r} != 'FMHA_TUNE_DBS' or 'double-buffered' in fm.kernel_for(L, N, h, d, fm.BF16 if td == torch.bfloat16 else fm.F16)\n"
        "    o, lse = fm.fmha_fwd(q, k, v)\n"
        f"    np.savez({str(tmp_path)!r} + f'/out{{n}}.npz', o=o.float().cpu().numpy(), lse=lse.cpu().numpy())\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, "-c", code], check=True, env=dict(os.environ, **{env: "1"}), cwd=root,
                   timeout=600)
    for n, (L, N, h, s) in enumerate(cases):
        q, k, v = probs[n]
        out = np.load(tmp_path / f"out{n}.npz")
        if N * h * L > 400 * 128:  # large case: a sample of Q tiles through the tile oracle
            tiles = [(b, hh, t) for b in range(L) for hh in (0, h // 2, h - 1) for t in (0, (N - 1) // 128)]
            o_ref, lse_ref = oracle.fmha_tiles(q, k, v, tiles, 128, 128)
            for ti, (b, hh, t) in enumerate(tiles):
                r0, r1 = t * 128, min(N, t * 128 + 128)
                res = errors(out["o"][b, r0:r1, hh], out["lse"][b, hh, r0:r1], o_ref[ti][: r1 - r0],
                             lse_ref[ti][: r1 - r0])
                assert_within(res, f"{env} {dt} L={L} N={N} h={h} tile {(b, hh, t)}")
        else:
            bm = 128 if N % 128 == 0 else N
            o_ref, lse_ref = oracle.fmha_forward(q, k, v, bm, bm)
            res = errors(out["o"], out["lse"], o_ref, lse_ref)
            assert_within(res, f"{env} {dt} L={L} N={N} h={h} scale {s}")
