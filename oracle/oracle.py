"""ctypes front-end for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Loads ``oracle/liboracle.so`` (the C restatement in ``fmha_oracle.c``) and,
when present, ``oracle/_ref/libfmhasim_ref.so`` (the reference compiled from
its own sources by ``oracle/Makefile``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs may import
this module; the product package never does.

All arrays are float32 BSHD ``(L, N, h, d)`` like the reference's ``Tensor4``
(``proj/include/fmhasim/tensor.hpp:12-32``); LSE is ``(L, h, N)`` float32.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libfmhasim_ref.so")

EXACT_F32 = 0
F16_EMU = 1
Q_F16 = 1
Q_BF16 = 2

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i64 = C.c_int64

_lib = None
_ref = None


def build():
    """Compile liboracle.so (and oracle/_ref when the reference is present)."""
    subprocess.check_call(["make", "-s", "-C", HERE, "all"])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.orc_gaussian_fill.argtypes = [_f32p, _i64, C.c_uint64]
        L.orc_quantize.argtypes = [_f32p, _i64, C.c_int]
        L.orc_to_half_bits.argtypes = [_f32p, _u16p, _i64, C.c_int]
        L.orc_from_half_bits.argtypes = [_u16p, _f32p, _i64, C.c_int]
        L.orc_f16_round.argtypes = [C.c_float]
        L.orc_f16_round.restype = C.c_float
        L.orc_bf16_round.argtypes = [C.c_float]
        L.orc_bf16_round.restype = C.c_float
        L.orc_default_scale.argtypes = [_i64]
        L.orc_default_scale.restype = C.c_float
        L.orc_validate.argtypes = [_i64] * 4
        L.orc_fmha_forward.argtypes = [_f32p, _f32p, _f32p] + [_i64] * 6 + [
            C.c_float, C.c_int, _f32p, C.c_void_p, C.c_int]
        L.orc_fmha_tiles.argtypes = [_f32p, _f32p, _f32p] + [_i64] * 6 + [
            C.c_float, C.c_int, _i64p, _i64, _f32p, _f32p, C.c_int]
        L.orc_standard_attention.argtypes = [_f32p, _f32p, _f32p] + [_i64] * 4 + [
            C.c_float, C.c_int, _f32p, C.c_void_p, C.c_int]
        L.orc_attention_flops.argtypes = [_i64] * 4
        L.orc_attention_flops.restype = _i64
        L.orc_fnv1a64.argtypes = [C.c_void_p, _i64]
        L.orc_fnv1a64.restype = C.c_uint64
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    """The reference itself (oracle/_ref), or None when it was not built."""
    global _ref
    if _ref is None and ref_available():
        R = C.CDLL(REF_PATH)
        R.ref_gaussian.argtypes = [_i64] * 4 + [C.c_uint64, _f32p]
        R.ref_f16_round.argtypes = [C.c_float]
        R.ref_f16_round.restype = C.c_float
        R.ref_fmha_forward.argtypes = [_f32p, _f32p, _f32p] + [_i64] * 6 + [C.c_int, _f32p]
        R.ref_standard_attention.argtypes = [_f32p, _f32p, _f32p] + [_i64] * 4 + [C.c_int, _f32p]
        R.ref_fmha_forward_heads.argtypes = [_f32p, _f32p, _f32p] + [_i64] * 5 + [_f32p, C.c_int]
        R.ref_fmha_tiles.argtypes = [_f32p, _f32p, _f32p] + [_i64] * 6 + [
            C.c_int, _i64p, _i64, _f32p, _f32p, C.c_int]
        R.ref_save_tensor.argtypes = [C.c_char_p, _f32p] + [_i64] * 4 + [C.c_int]
        R.ref_load_tensor.argtypes = [C.c_char_p, _f32p, _i64, _i64p]
        _ref = R
    return _ref


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


# ----------------------------------------------------------------- inputs --
def gaussian(L, N, h, d, seed) -> np.ndarray:
    """gaussian_tensor(L,N,h,d,seed), random.hpp:44-50."""
    out = np.empty((L, N, h, d), np.float32)
    lib().orc_gaussian_fill(out.reshape(-1), out.size, seed)
    return out


def quantize(x: np.ndarray, dtype: str) -> np.ndarray:
    """Round float32 to f16 (reference f16_round semantics) or bf16 (RNE)."""
    y = np.ascontiguousarray(x, np.float32).copy()
    lib().orc_quantize(y.reshape(-1), y.size, Q_F16 if dtype == "f16" else Q_BF16)
    return y


def to_bits(x: np.ndarray, dtype: str) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty(x.shape, np.uint16)
    lib().orc_to_half_bits(x.reshape(-1), out.reshape(-1), x.size, Q_F16 if dtype == "f16" else Q_BF16)
    return out


def from_bits(b: np.ndarray, dtype: str) -> np.ndarray:
    b = np.ascontiguousarray(b, np.uint16)
    out = np.empty(b.shape, np.float32)
    lib().orc_from_half_bits(b.reshape(-1), out.reshape(-1), b.size, Q_F16 if dtype == "f16" else Q_BF16)
    return out


def problem(L, N, h, d, seed=42, dtype=None):
    """Q, K, V from seeds (seed, seed+1, seed+2) as fmha_cli.cpp:79-84, optionally
    quantised to the GPU's 16-bit input type."""
    qkv = [gaussian(L, N, h, d, seed + i) for i in range(3)]
    if dtype is not None:
        qkv = [quantize(t, dtype) for t in qkv]
    return qkv


def default_scale(d) -> float:
    return float(lib().orc_default_scale(d))


# ------------------------------------------------------------------ math --
def fmha_forward(q, k, v, bM=64, bN=64, prec=EXACT_F32, scale=None, threads=None, want_lse=True):
    """fmha_forward (attention.cpp:153-173) + LSE; returns (O, lse)."""
    L, N, h, d = q.shape
    scale = default_scale(d) if scale is None else scale
    O = np.empty_like(q)
    lse = np.empty((L, h, N), np.float32) if want_lse else None
    st = lib().orc_fmha_forward(q, k, v, L, N, h, d, bM, bN, scale, prec, O,
                                lse.ctypes.data if want_lse else None, threads or default_threads())
    if st:
        raise ValueError(f"TileConfig: N = {N} must be divisible by bM = {bM} and bN = {bN}")
    return O, lse


def standard_attention(q, k, v, prec=EXACT_F32, scale=None, threads=None):
    L, N, h, d = q.shape
    scale = default_scale(d) if scale is None else scale
    O = np.empty_like(q)
    lse = np.empty((L, h, N), np.float32)
    lib().orc_standard_attention(q, k, v, L, N, h, d, scale, prec, O, lse.ctypes.data,
                                 threads or default_threads())
    return O, lse


def fmha_tiles(q, k, v, tiles, bM=128, bN=128, prec=EXACT_F32, scale=None, threads=None):
    """O (n, bM, d) and LSE (n, bM) for the listed (b, head, i) Q tiles."""
    L, N, h, d = q.shape
    scale = default_scale(d) if scale is None else scale
    t = np.ascontiguousarray(np.asarray(tiles, np.int64).reshape(-1, 3))
    O = np.empty((len(t), bM, d), np.float32)
    lse = np.empty((len(t), bM), np.float32)
    st = lib().orc_fmha_tiles(q, k, v, L, N, h, d, bM, bN, scale, prec, t.reshape(-1), len(t), O, lse,
                              threads or default_threads())
    if st:
        raise ValueError("invalid tiling or tile index")
    return O, lse


def attention_flops(L, N, h, d) -> int:
    return int(lib().orc_attention_flops(L, N, h, d))


def fnv1a64(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return "%016x" % lib().orc_fnv1a64(a.ctypes.data, a.nbytes)


# ------------------------------------------------- reference passthrough --
def ref_gaussian(L, N, h, d, seed):
    out = np.empty((L, N, h, d), np.float32)
    ref().ref_gaussian(L, N, h, d, seed, out.reshape(-1))
    return out


def ref_fmha_forward(q, k, v, bM=64, bN=64, prec=EXACT_F32):
    L, N, h, d = q.shape
    out = np.empty_like(q)
    if ref().ref_fmha_forward(q, k, v, L, N, h, d, bM, bN, prec, out):
        raise ValueError("invalid tiling")
    return out


def ref_standard_attention(q, k, v, prec=EXACT_F32):
    L, N, h, d = q.shape
    out = np.empty_like(q)
    ref().ref_standard_attention(q, k, v, L, N, h, d, prec, out)
    return out


def ref_fmha_tiles(q, k, v, tiles, bM=128, bN=128, prec=EXACT_F32, threads=None):
    L, N, h, d = q.shape
    t = np.ascontiguousarray(np.asarray(tiles, np.int64).reshape(-1, 3))
    O = np.empty((len(t), bM, d), np.float32)
    lse = np.empty((len(t), bM), np.float32)
    if ref().ref_fmha_tiles(q, k, v, L, N, h, d, bM, bN, prec, t.reshape(-1), len(t), O, lse,
                            threads or default_threads()):
        raise ValueError("invalid tiling")
    return O, lse


def ref_fmha_forward_heads(qh, kh, vh, bM=128, bN=128, threads=None):
    """Reference fmha_forward over packed single heads (heads, N, d), threaded."""
    H, N, d = qh.shape
    out = np.empty_like(qh)
    ref().ref_fmha_forward_heads(qh, kh, vh, H, N, d, bM, bN, out, threads or default_threads())
    return out


def ref_save_tensor(path, t, f16=False):
    t = np.ascontiguousarray(t, np.float32)
    L, N, h, d = t.shape
    return ref().ref_save_tensor(path.encode(), t.reshape(-1), L, N, h, d, int(f16))


def ref_load_tensor(path, capacity=1 << 24):
    out = np.empty(capacity, np.float32)
    dims = np.zeros(4, np.int64)
    st = ref().ref_load_tensor(path.encode(), out, capacity, dims)
    if st:
        raise RuntimeError("reference load_tensor failed")
    L, N, h, d = (int(x) for x in dims)
    return out[: L * N * h * d].reshape(L, N, h, d).copy()
