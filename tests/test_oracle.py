"""The CPU oracle (oracle/fmha_oracle.c) pinned against the reference.

* golden hashes recorded from the REFERENCE build (tests/golden/goldens.json,
  made by tests/golden/make_goldens.py from oracle/_ref, and identical to
  SURVEY.md Appendix A);
* bit-exact comparison with oracle/_ref itself when it is built here;
* the reference's own known-answer and property tests for this path
  (proj/tests/test_attention.cpp, acceptance.cpp criteria 3/4/8,
  test_io.cpp), restated against the oracle.
"""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLD, "goldens.json")) as f:
        return json.load(f)


def test_gaussian_fixture_hashes(oracle, gold):
    """gaussian_tensor(1,512,1,64,seed) (random.hpp:44-50), seeds 42/43/44."""
    for s, h in gold["gaussian_1_512_1_64"].items():
        assert oracle.fnv1a64(oracle.gaussian(1, 512, 1, 64, int(s))) == h
    np.testing.assert_array_equal(oracle.gaussian(1, 512, 1, 64, 42).reshape(-1)[:3],
                                  np.array(gold["gaussian_first3_seed42"], np.float32))


def test_config1_fmha_hashes(oracle, gold):
    """fmha_forward on config 1, both tilings and both precisions, bitwise."""
    q, k, v = oracle.problem(1, 512, 1, 64, 42)
    for bm in (64, 128):
        for prec, name in ((oracle.EXACT_F32, "f32"), (oracle.F16_EMU, "f16emu")):
            o, _ = oracle.fmha_forward(q, k, v, bm, bm, prec=prec)
            assert oracle.fnv1a64(o) == gold["c1_fmha"][f"{bm}x{bm}_{name}"], (bm, name)
    o, _ = oracle.standard_attention(q, k, v)
    assert oracle.fnv1a64(o) == gold["c1_standard_f32"]
    qq, kk, vv = (oracle.quantize(x, "f16") for x in (q, k, v))
    assert oracle.fnv1a64(oracle.fmha_forward(qq, kk, vv, 64, 64)[0]) == gold["c1_f16inputs_64x64_f32"]


def test_survey_appendix_a_hashes(oracle):
    """The same values as SURVEY.md Appendix A (recorded independently)."""
    q, k, v = oracle.problem(1, 512, 1, 64, 42)
    assert oracle.fnv1a64(q) == "3bdf938039f36926"
    assert oracle.fnv1a64(oracle.fmha_forward(q, k, v, 64, 64)[0]) == "52f88399bc48e4fa"
    assert oracle.fnv1a64(oracle.fmha_forward(q, k, v, 64, 64, prec=oracle.F16_EMU)[0]) == "7c64b8816f70296e"
    assert oracle.fnv1a64(oracle.gaussian(1, 512, 1, 64, 1060)) == "4f82d92d80cbba21"


def test_acceptance_c3_grid_hashes(oracle, gold):
    """acceptance.cpp:71-96 grid: 9 (N, d) pairs x 4 tilings, bitwise to the reference."""
    grid = gold["acceptance_c3_grid"]
    seed = 1000
    for N in (128, 256, 512):
        for d in (64, 128, 256):
            q, k, v = (oracle.gaussian(1, N, 1, d, seed + i) for i in range(3))
            for bm in (64, 128):
                for bn in (64, 128):
                    o, _ = oracle.fmha_forward(q, k, v, bm, bn, want_lse=False)
                    assert oracle.fnv1a64(o) == grid[f"N{N}_d{d}_{bm}x{bn}_seed{seed}"]
            seed += 10


def test_acceptance_c3_tolerance(oracle):
    """Fused vs standard <= 1e-5 under |a-b|/max(|b|,1) (acceptance.cpp:71-96)."""
    q, k, v = oracle.problem(1, 256, 1, 128, 1010)
    ref, _ = oracle.standard_attention(q, k, v)
    for bm in (64, 128):
        for bn in (64, 128):
            o, _ = oracle.fmha_forward(q, k, v, bm, bn)
            assert (np.abs(o - ref) / np.maximum(np.abs(ref), 1)).max() <= 1e-5


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(GOLD), "..", "oracle", "_ref",
                                                    "libfmhasim_ref.so")), reason="oracle/_ref not built")
def test_bitwise_equal_to_reference_build(oracle):
    """The restatement equals the reference compiled from its own sources."""
    for (L, N, h, d, bm, bn, prec) in [(2, 128, 3, 32, 64, 32, 0), (1, 256, 2, 64, 128, 64, 0),
                                       (1, 128, 1, 64, 64, 64, 1)]:
        q, k, v = oracle.problem(L, N, h, d, 5 + N)
        o, lse = oracle.fmha_forward(q, k, v, bm, bn, prec=prec)
        np.testing.assert_array_equal(o, oracle.ref_fmha_forward(q, k, v, bm, bn, prec))
        tiles = [(b, hh, i) for b in range(L) for hh in range(h) for i in range(N // bm)]
        o_t, lse_t = oracle.ref_fmha_tiles(q, k, v, tiles, bm, bn, prec)
        np.testing.assert_array_equal(lse_t.reshape(L, h, N), lse)
    np.testing.assert_array_equal(oracle.ref_gaussian(2, 16, 3, 8, 99), oracle.gaussian(2, 16, 3, 8, 99))
    xs = np.random.default_rng(1).standard_normal(10000).astype(np.float32) * 1e3
    for x in xs[:2000]:
        assert oracle.ref().ref_f16_round(float(x)) == oracle.lib().orc_f16_round(float(x))


def test_scalar_problem(oracle):
    """test_attention.cpp:69-77: N = d = 1, O == input."""
    x = np.full((1, 1, 1, 1), 0.7, np.float32)
    o, lse = oracle.fmha_forward(x, x, x, 1, 1)
    assert o[0, 0, 0, 0] == np.float32(0.7)
    assert lse[0, 0, 0] == np.float32(0.7) * np.float32(0.7)  # s*scale with scale = 1, ln(1) = 0


def test_single_tile_fused_equals_standard_bitwise(oracle):
    """test_attention.cpp:143-148."""
    q, k, v = oracle.problem(2, 64, 2, 32, 41)
    np.testing.assert_array_equal(oracle.fmha_forward(q, k, v, 64, 64)[0], oracle.standard_attention(q, k, v)[0])


def test_tile_indivisibility_rejected(oracle):
    """test_attention.cpp:159-164."""
    q, k, v = oracle.problem(1, 96, 1, 16, 2)
    for bm, bn in ((64, 32), (32, 64), (128, 32)):
        with pytest.raises(ValueError):
            oracle.fmha_forward(q, k, v, bm, bn)


def test_dense_double_oracle(oracle):
    """standard attention vs an independent float64 dense oracle (test_attention.cpp:19-50,96-99)."""
    q, k, v = oracle.problem(1, 128, 1, 64, 17)
    o, lse = oracle.standard_attention(q, k, v)
    Q, K, V = (t[0, :, 0].astype(np.float64) for t in (q, k, v))
    S = Q @ K.T / np.sqrt(64.0)
    m = S.max(axis=1, keepdims=True)
    P = np.exp(S - m)
    ref = (P / P.sum(axis=1, keepdims=True)) @ V
    assert (np.abs(o[0, :, 0] - ref) / np.maximum(np.abs(ref), 1)).max() <= 1e-6
    np.testing.assert_allclose(lse[0, 0], (m[:, 0] + np.log(P.sum(axis=1))), rtol=1e-6)


def test_flops(oracle):
    """acceptance.cpp:215-223 (criterion 8): spot value 16,777,216."""
    assert oracle.attention_flops(1, 256, 1, 64) == 16777216
    assert oracle.attention_flops(8, 16384, 32, 128) == 35184372088832


def test_half_rounding_kats(oracle):
    """test_attention.cpp:290-299 and test_io.cpp:28-37."""
    r = oracle.lib().orc_f16_round
    assert r(1.0) == 1.0
    assert r(0.1) == np.float32(0.0999755859375)
    assert r(-2.5) == -2.5
    assert r(1e6) == 65504.0 and r(-1e6) == -65504.0
    assert abs(r(6e-5) - 6e-5) / 6e-5 < 1e-3
    assert oracle.lib().orc_bf16_round(1.0) == 1.0
    assert oracle.lib().orc_bf16_round(1.00390625) == 1.0  # tie to even
    assert oracle.lib().orc_bf16_round(1.01171875) == np.float32(1.015625)


def test_seed_determinism(oracle):
    """test_io.cpp:61-76."""
    a = oracle.gaussian(1, 8, 2, 4, 1234)
    assert np.array_equal(a, oracle.gaussian(1, 8, 2, 4, 1234))
    assert not np.array_equal(a, oracle.gaussian(1, 8, 2, 4, 1235))


def test_bshd_offsets():
    """test_io.cpp:52-59: offset(b,n,head,k) = n*d*h + k + head*d + b*h*N*d."""
    L, N, h, d = 2, 4, 3, 5
    idx = np.arange(L * N * h * d).reshape(L, N, h, d)
    assert idx[0, 0, 0, 1] == 1 and idx[0, 0, 1, 0] == 5 and idx[0, 1, 0, 0] == 15
    assert idx[1, 0, 0, 0] == 3 * 4 * 5


def test_sampled_tiles_match_full_run(oracle):
    """Sub-problem sampling is bitwise identical to the full run."""
    q, k, v = oracle.problem(2, 256, 3, 64, 8)
    o, lse = oracle.fmha_forward(q, k, v, 128, 128)
    tiles = [(1, 2, 1), (0, 0, 0)]
    o_t, lse_t = oracle.fmha_tiles(q, k, v, tiles, 128, 128)
    np.testing.assert_array_equal(o_t[0], o[1, 128:256, 2])
    np.testing.assert_array_equal(lse_t[1], lse[0, 0, :128])
    # one head sliced out and run alone
    oh, _ = oracle.fmha_forward(*(np.ascontiguousarray(t[1:2, :, 2:3]) for t in (q, k, v)), 128, 128)
    np.testing.assert_array_equal(oh[0, :, 0], o[1, :, 2])


def test_stream_equivalence(oracle):
    """Online softmax == one-shot over random tilings, restated through the
    oracle's tiled path: different bN must give LSE equal within 1e-6
    (acceptance.cpp:99-123, test_attention.cpp:166-192)."""
    q, k, v = oracle.problem(1, 512, 2, 64, 2024)
    _, l0 = oracle.standard_attention(q, k, v)
    for bn in (1, 7 * 0 + 8, 64, 128, 256):
        _, l1 = oracle.fmha_forward(q, k, v, 128, bn)
        assert np.abs((l1 - l0) / l0).max() <= 1e-6
