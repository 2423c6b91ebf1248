"""The C-ABI library on CPU: it loads, exports every symbol include/fmha/fmha.h
declares, validates arguments like the reference (attention.cpp:13-27), and its
host-side 16-bit converters agree with the reference quantiser.  No kernel is
launched here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2312_11918_b200 as fm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "fmha", "fmha.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b([a-z_0-9]+)\s*\(", src)
    return sorted({n for n in names if n.startswith("fmha_")})


def test_library_exports_every_declared_symbol():
    lib = fm.lib()
    names = declared_functions()
    assert {"fmha_fwd", "fmha_fwd_check", "fmha_fwd_host", "fmha_forward_f32", "fmha_last_error"} <= set(names)
    for n in names:
        assert hasattr(lib, n), f"{n} declared in fmha.h but not exported"


def test_sm100a_code_present():
    """The library carries sm_100a SASS with tcgen05 / TMA instructions."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-sass", fm.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for mnem in ("UTCHMMA", "UTMALDG", "LDTM", "STTM"):
        assert mnem in out, mnem
    assert "HMMA" not in out.replace("UTCHMMA", ""), "legacy mma.sync path present"


def test_version_and_flops():
    assert b"sm_100a" in fm.lib().fmha_version()
    assert fm.attention_flops(1, 256, 1, 64) == 16777216
    assert fm.attention_flops(4, 4096, 16, 128) == 549755813888


def _check(p):
    return fm.lib().fmha_fwd_check(C.byref(p))


def test_check_validation():
    p = fm.dense_params(4, 4096, 16, 128, fm.F16)
    assert _check(p) == fm.OK
    for d in (64, 256):
        assert _check(fm.dense_params(1, 512, 1, d)) == fm.OK
    # what the reference rejects (attention.cpp:16-17)
    assert _check(fm.dense_params(1, 0, 1, 64)) == fm.ERR_CONFIG
    assert b"N >= 1" in fm.lib().fmha_last_error()
    assert _check(fm.dense_params(1, 16, 1, 0)) == fm.ERR_CONFIG
    # valid for the reference, not for the tensor-core kernel
    assert _check(fm.dense_params(1, 16, 1, 32)) == fm.ERR_UNSUPPORTED
    # TMA needs 16-B aligned strides
    p = fm.dense_params(1, 64, 3, 64)
    p.k_stride[1] = 100
    assert _check(p) == fm.ERR_CONFIG
    p = fm.dense_params(1, 64, 1, 64)
    p.dtype = 7
    assert _check(p) == fm.ERR_CONFIG
    # grid limits: h, L <= 65535 and < 2^31 work units of 256 query rows
    assert _check(fm.dense_params(1, 256, 65536, 64)) == fm.ERR_UNSUPPORTED
    assert _check(fm.dense_params(65535, 1 << 24, 65535, 64)) == fm.ERR_UNSUPPORTED
    assert b"work units" in fm.lib().fmha_last_error()


def test_fwd_rejects_null_before_launch():
    p = fm.dense_params(1, 128, 1, 64)
    st = fm.lib().fmha_fwd(C.byref(p), None, None, None, None, None, None)
    assert st == fm.ERR_CONFIG


def test_python_front_end_errors():
    q = np.zeros((1, 100, 1, 64), np.float32)
    with pytest.raises(ValueError, match="divisible"):
        fm.fmha_forward(q, q, q, 64, 64)  # bindings.cpp / test_smoke.py:43-46
    with pytest.raises(ValueError, match="16-bit"):
        fm.fmha_forward(q, q, q, 100, 100, precision="f32")
    with pytest.raises(ValueError, match="shape"):
        fm.fmha_forward(q, q[:, :50], q, 50, 50)
    with pytest.raises(ValueError):
        fm.fmha_forward(np.zeros((1, 64, 1, 32), np.float32), *([np.zeros((1, 64, 1, 32), np.float32)] * 2), 64, 64)


def test_host_f16_conversion_matches_reference_quantiser(oracle):
    """fmha_forward_f32 quantises with the reference's f16 semantics
    (RNE, saturating, subnormals kept: half.hpp:12-42)."""
    lib = fm.lib()
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.standard_normal(20000) * s for s in (1e-7, 1e-5, 1e-3, 1, 100, 1e4, 1e5)]).astype(np.float32)
    edge = np.array([0.0, -0.0, 65504, 65519.99, 65520, 65536, 1e30, -1e30, 2 ** -24, 2 ** -25,
                     1.5 * 2 ** -25, 2 ** -14, 2 ** -14 * (1 - 2 ** -12), 6e-5, 0.1, np.inf, -np.inf], np.float32)
    xs = np.concatenate([xs, edge])
    ref_bits = oracle.to_bits(xs, "f16")
    got = np.array([lib.fmha_host_f32_to_16(float(x), 0) for x in xs], np.uint16)
    np.testing.assert_array_equal(got, ref_bits)
    back = np.array([lib.fmha_host_16_to_f32(int(b), 0) for b in ref_bits], np.float32)
    np.testing.assert_array_equal(back, oracle.from_bits(ref_bits, "f16"))
    ref_bf = oracle.to_bits(xs, "bf16")
    got_bf = np.array([lib.fmha_host_f32_to_16(float(x), 1) for x in xs], np.uint16)
    np.testing.assert_array_equal(got_bf, ref_bf)
    nan16 = lib.fmha_host_f32_to_16(float("nan"), 0)
    assert (nan16 & 0x7C00) == 0x7C00 and (nan16 & 0x3FF) != 0


def test_bulk_quantiser_matches_elementwise(oracle):
    """fmha_host_quantize / dequantize (threaded, F16C fast path) are bit-identical
    to the reference quantiser on ordinary values and on every special case
    (saturation band, inf, NaN, subnormals), including odd lengths and tails."""
    import ctypes as C
    lib = fm.lib()
    lib.fmha_host_quantize.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int]
    lib.fmha_host_dequantize.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int]
    rng = np.random.default_rng(1)
    xs = np.concatenate([rng.standard_normal(300001) * s for s in (1e-7, 1e-4, 1, 3e4, 1e5)]).astype(np.float32)
    special = np.array([65504, 65519.99, 65520, -65520, 7e4, np.inf, -np.inf, np.nan, 2 ** -24, 2 ** -25,
                        1.5 * 2 ** -25, -0.0, 2 ** -14 * (1 - 2 ** -12)], np.float32)
    xs[rng.integers(0, xs.size, 5000)] = rng.choice(special, 5000)
    for dt, code in (("f16", fm.F16), ("bf16", fm.BF16)):
        got = np.empty(xs.size, np.uint16)
        lib.fmha_host_quantize(xs.ctypes.data, got.ctypes.data, xs.size, code)
        ref = oracle.to_bits(xs, dt)
        nan = np.isnan(xs)
        np.testing.assert_array_equal(got[~nan], ref[~nan])
        assert np.all((got[nan] & 0x7F80 if dt == "bf16" else got[nan] & 0x7C00) > 0)
        back = np.empty(xs.size, np.float32)
        lib.fmha_host_dequantize(got.ctypes.data, back.ctypes.data, xs.size, code)
        np.testing.assert_array_equal(back[~nan], oracle.from_bits(got, dt)[~nan])


def test_cpp_adapter_header_compiles(tmp_path):
    """The C++ drop-in adapter header (fmha.hpp) compiles against a reference-style caller."""
    import shutil
    import subprocess
    if not shutil.which("g++"):
        pytest.skip("no g++")
    src = tmp_path / "caller.cpp"
    src.write_text('''
#include "fmha/fmha.hpp"
int main() {
  using namespace fmha_b200;
  Tensor4 q(1, 128, 2, 64), k(1, 128, 2, 64), v(1, 128, 2, 64);
  AttentionProblem p(q, k, v);
  validate_tiling(p, TileConfig{64, 64});
  try { validate_tiling(p, TileConfig{96, 64}); return 1; } catch (const std::invalid_argument&) {}
  try { fmha_forward(p, TileConfig{64, 64}, Precision::ExactF32); return 2; } catch (const std::invalid_argument&) {}
  return attention_flops(1, 256, 1, 64) == 16777216 ? 0 : 3;
}
''')
    exe = tmp_path / "caller"
    subprocess.check_call(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                           fm.LIB_PATH, f"-Wl,-rpath,{os.path.dirname(fm.LIB_PATH)}"])
    assert subprocess.run([str(exe)]).returncode == 0
