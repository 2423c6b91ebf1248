"""GPU parity of the drop-in entry points that take the reference's own call
shape (float host Tensor4 in and out, copies and 16-bit quantisation inside):

* the C++ adapter ``fmha_b200::fmha_forward(AttentionProblem, TileConfig,
  Precision[, &lse])`` (include/fmha/fmha.hpp, replacing
  /root/reference/proj/include/fmhasim/attention.hpp:58-59), driven by a
  reference-style C++ caller compiled here against the header and the
  in-tree library -- over the reference's acceptance grid
  (/root/reference/proj/tests/acceptance.cpp:71-96: N in {128,256,512} x
  d in {64,128,256}, seeds 1000 + 10k, every (bM, bN) in {64,128}^2), for
  F16Emu and BF16, with and without LSE, and at config 3 with the
  reference's seeds 42/43/44 (sampled Q tiles);
* the Python ``fmha_forward`` (the pybind call shape, bindings.cpp:81-91) over
  ``fmha_forward_f32`` at config 3 (fp16) and config 5 (bf16) sizes, where
  the host pipeline quantises per input chunk and slices the last batch by
  query rows.

The oracle (oracle/fmha_oracle.c, pinned to the reference build) runs on the
same 16-bit-rounded inputs; tolerances are the north-star ones (parity.py).
"""
import os
import shutil
import subprocess

import numpy as np
import pytest

from parity import assert_within, errors

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CALLER = r'''
// A reference-style caller: fmhasim:: -> fmha_b200::, include swapped, the
// rest is the reference's call shape (attention.hpp:14-30, :58-59).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include "fmha/fmha.hpp"
int main(int argc, char** argv) {
  using namespace fmha_b200;
  int failures = 0;
  for (int i = 1; i < argc; ++i) {
    const std::string dir = argv[i];
    std::ifstream pf(dir + "/params.txt");
    std::string prec;
    int want_lse = 0;
    long long bM = 0, bN = 0;
    pf >> prec >> want_lse >> bM >> bN;
    try {
      AttentionProblem p(load_tensor(dir + "/q.fhmt"), load_tensor(dir + "/k.fhmt"), load_tensor(dir + "/v.fhmt"));
      const Precision pr = prec == "bf16" ? Precision::BF16 : prec == "f32" ? Precision::ExactF32 : Precision::F16Emu;
      std::vector<float> lse;
      Tensor4 o = want_lse ? fmha_forward(p, TileConfig{bM, bN}, pr, &lse) : fmha_forward(p, TileConfig{bM, bN}, pr);
      save_tensor(o, dir + "/o.fhmt");
      if (want_lse) {
        Tensor4 l(p.L(), p.heads(), p.N(), 1);
        l.data = lse;
        save_tensor(l, dir + "/lse.fhmt");
      }
      std::ofstream(dir + "/status.txt") << "ok\n";
    } catch (const std::invalid_argument& e) {
      std::ofstream(dir + "/status.txt") << "invalid_argument " << e.what() << "\n";
    } catch (const std::exception& e) {
      std::ofstream(dir + "/status.txt") << "error " << e.what() << "\n";
      ++failures;
    }
  }
  return failures;
}
'''


@pytest.fixture(scope="module")
def caller(tmp_path_factory):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not shutil.which("g++"):
        pytest.skip("no g++")
    import paper_2312_11918_b200 as fm
    d = tmp_path_factory.mktemp("caller")
    (d / "caller.cpp").write_text(CALLER)
    exe = d / "caller"
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), str(d / "caller.cpp"),
                           "-o", str(exe), fm.LIB_PATH, f"-Wl,-rpath,{os.path.dirname(fm.LIB_PATH)}"])
    return str(exe)


def _write_case(fm, d, q, k, v, prec, want_lse, bM, bN, file_prec="f32"):
    d.mkdir(parents=True, exist_ok=True)
    for name, t in (("q", q), ("k", k), ("v", v)):
        fm.save_tensor(t, d / f"{name}.fhmt", precision=file_prec)
    (d / "params.txt").write_text(f"{prec} {int(want_lse)} {bM} {bN}\n")


def _run(caller, dirs):
    r = subprocess.run([caller] + [str(x) for x in dirs], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr + "".join((x / "status.txt").read_text() for x in dirs
                                                            if (x / "status.txt").exists())


def test_cpp_adapter_acceptance_grid(oracle, caller, tmp_path):
    """acceptance.cpp:71-96's grid through the C++ drop-in, F16Emu and BF16,
    with and without LSE, every tiling the reference sweeps (the tiling is a
    validation contract here: the kernel picks its own tile shape)."""
    import paper_2312_11918_b200 as fm
    cases = []
    seed = 1000
    for N in (128, 256, 512):
        for d in (64, 128, 256):
            q, k, v = oracle.problem(1, N, 1, d, seed)  # gaussian_problem(1, N, 1, d, seed)
            seed += 10
            for i, (bM, bN) in enumerate([(64, 64), (64, 128), (128, 64), (128, 128)]):
                prec = "f16" if i % 2 == 0 else "bf16"
                want_lse = i < 2
                cdir = tmp_path / f"N{N}_d{d}_{bM}x{bN}"
                _write_case(fm, cdir, q, k, v, prec, want_lse, bM, bN)
                cases.append((cdir, q, k, v, prec, want_lse, N, d))
    _run(caller, [c[0] for c in cases])
    for cdir, q, k, v, prec, want_lse, N, d in cases:
        assert (cdir / "status.txt").read_text().startswith("ok"), (cdir / "status.txt").read_text()
        qq, kk, vv = (oracle.quantize(x, prec) for x in (q, k, v))  # the adapter's RNE rounding
        o_ref, lse_ref = oracle.fmha_forward(qq, kk, vv, 128 if N % 128 == 0 else N, 128 if N % 128 == 0 else N)
        o = fm.load_tensor(cdir / "o.fhmt")
        lse = fm.load_tensor(cdir / "lse.fhmt").reshape(1, 1, N) if want_lse else None
        assert not (cdir / "lse.fhmt").exists() or want_lse
        assert_within(errors(o, lse, o_ref, lse_ref if want_lse else None), f"C++ adapter {cdir.name} {prec}")


def test_cpp_adapter_rejections(oracle, caller, tmp_path):
    """What the reference rejects with std::invalid_argument (tile
    indivisibility, attention.cpp:21-27) and what the GPU path rejects
    (ExactF32: no fp32 / CPU fallback) surface as std::invalid_argument."""
    import paper_2312_11918_b200 as fm
    q, k, v = oracle.problem(1, 192, 1, 64, 5)
    bad_tile = tmp_path / "bad_tile"
    _write_case(fm, bad_tile, q, k, v, "f16", True, 128, 64)  # 192 % 128 != 0
    exact = tmp_path / "exact"
    _write_case(fm, exact, q, k, v, "f32", False, 64, 64)
    _run(caller, [bad_tile, exact])
    assert (bad_tile / "status.txt").read_text().startswith("invalid_argument")
    assert "divisible" in (bad_tile / "status.txt").read_text()
    assert (exact / "status.txt").read_text().startswith("invalid_argument")
    assert not (bad_tile / "o.fhmt").exists()


def _sample_check(oracle, o, lse, q, k, v, heads, n_tiles, rng, ctx):
    for (b, hh) in heads:
        qh, kh, vh = (np.ascontiguousarray(x[b:b + 1, :, hh:hh + 1, :]) for x in (q, k, v))
        tiles = sorted({0, n_tiles - 1, int(rng.integers(n_tiles))})
        o_ref, lse_ref = oracle.fmha_tiles(qh, kh, vh, [(0, 0, i) for i in tiles], 128, 128)
        o_got = np.stack([o[b, i * 128:(i + 1) * 128, hh] for i in tiles])
        lse_got = np.stack([lse[b, hh, i * 128:(i + 1) * 128] for i in tiles]) if lse is not None else None
        assert_within(errors(o_got, lse_got, o_ref, lse_ref if lse is not None else None),
                      f"{ctx} b={b} h={hh} tiles={tiles}")


def test_cpp_adapter_config3_reference_seeds(oracle, caller, tmp_path):
    """Config 3 (L=4, h=16, N=4096, d=128) with the reference's own inputs
    (gaussian_tensor seeds 42/43/44, fmha_cli.cpp:79-84) through the C++
    drop-in with LSE; sampled Q tiles of the first / middle / last batch."""
    import paper_2312_11918_b200 as fm
    L, N, h, d = 4, 4096, 16, 128
    q, k, v = oracle.problem(L, N, h, d, 42, dtype="f16")  # f16-exact, so f16 fixture files are lossless
    cdir = tmp_path / "c3"
    _write_case(fm, cdir, q, k, v, "f16", True, 128, 128, file_prec="f16")
    _run(caller, [cdir])
    o = fm.load_tensor(cdir / "o.fhmt")
    lse = fm.load_tensor(cdir / "lse.fhmt").reshape(L, h, N)
    heads = [(b, hh) for b in (0, L // 2, L - 1) for hh in (0, h - 1)]
    _sample_check(oracle, o, lse, q, k, v, heads, N // 128, np.random.default_rng(3), "C++ adapter c3")
    assert np.isfinite(o).all() and np.isfinite(lse).all()


def _float_path_case(oracle, L, N, h, d, prec, seed):
    """Python fmha_forward (fmha_forward_f32): float32 host arrays in and out."""
    import paper_2312_11918_b200 as fm
    rng = np.random.default_rng(seed)
    q, k, v = (rng.standard_normal((L, N, h, d), dtype=np.float32) for _ in range(3))
    o, lse = fm.fmha_forward(q, k, v, 128, 128, precision=prec, return_lse=True)
    assert o.dtype == np.float32 and o.shape == q.shape and lse.shape == (L, h, N)
    dt = "bf16" if prec == "bf16" else "f16"
    heads = [(b, hh) for b in sorted({0, L // 2, L - 1}) for hh in (0, h - 1)]
    # the oracle sees the same RNE-rounded values the adapter fed the GPU
    qq, kk, vv = (oracle.quantize(np.ascontiguousarray(x[:, :, sorted({0, h - 1})]), dt) for x in (q, k, v))
    hmap = {hh: i for i, hh in enumerate(sorted({0, h - 1}))}
    o_s = o[:, :, sorted({0, h - 1})]
    lse_s = lse[:, sorted({0, h - 1})]
    _sample_check(oracle, o_s, lse_s, qq, kk, vv, [(b, hmap[hh]) for b, hh in heads], N // 128,
                  np.random.default_rng(seed + 1), f"fmha_forward_f32 L={L} N={N} h={h} d={d} {prec}")
    assert np.isfinite(o).all() and np.isfinite(lse).all()


def test_float_path_config3_f16(oracle):
    """Config 3 through the float call shape: 400 MB of float inputs, so the
    pipeline quantises per input chunk and slices the last batch by rows."""
    _float_path_case(oracle, 4, 4096, 16, 128, "f16emu", 31)


def test_float_path_config5_bf16(oracle):
    """Config 5 (L=8, h=32, N=16384, d=128, bf16) through the float call
    shape: 6.4 GB of float inputs on the host."""
    psutil = pytest.importorskip("psutil")
    need = 8 * 536870912 * 4 * 1.6  # q, k, v, o float32 + pinned 16-bit staging
    if psutil.virtual_memory().available < need:
        pytest.skip(f"needs {need / 2**30:.0f} GiB of host memory")
    _float_path_case(oracle, 8, 16384, 32, 128, "bf16", 47)


def test_two_devices_in_one_process():
    """Per-device state (shared-memory opt-in, SM count, workspaces): the host
    entry point on device 1 after device 0 in one process."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import paper_2312_11918_b200 as fm
    L, N, h, d = 1, 1024, 2, 128
    rng = np.random.default_rng(0)
    q, k, v = (rng.standard_normal((L, N, h, d), dtype=np.float32) for _ in range(3))
    o0 = fm.fmha_forward(q, k, v, 128, 128, device=0)
    o1 = fm.fmha_forward(q, k, v, 128, 128, device=1)
    np.testing.assert_array_equal(o0, o1)
    for dev in (0, 1):
        tq, tk, tv = (torch.from_numpy(x).to(f"cuda:{dev}").half() for x in (q, k, v))
        o, _ = fm.fmha_fwd(tq, tk, tv)
        torch.cuda.synchronize(dev)
        assert torch.isfinite(o.float()).all()
