"""paper_2312_11918_b200 -- B200-native (sm_100a) FMHA forward pass.

Python mirror of the reference's pybind entry point
``_fmhasim.fmha_forward(q, k, v, bM=64, bN=64, precision="f32")``
(/root/reference/proj/src/bindings.cpp:81-91) on top of the C ABI in
``include/fmha/fmha.h`` (loaded with ctypes from the in-tree
``libfmha_b200.so``).  There is no CPU fallback: if the library or a GPU is
missing, calls fail loudly.

Three entry points:

* :func:`fmha_forward` -- reference call shape: float32 numpy BSHD arrays in,
  float32 out; ``precision`` is ``"f16emu"``/``"f16"`` or ``"bf16"``
  (``"f32"`` raises ``ValueError``: the GPU path is 16-bit); invalid tiling
  raises ``ValueError`` exactly like the reference (``test_smoke.py:43-46``).
* :func:`fmha_fwd` -- device tensors (torch CUDA, fp16/bf16, BSHD with any
  16-B aligned strides), asynchronous on the current stream, optional LSE.
* :func:`fmha_fwd_host` -- host 16-bit buffers in/out (copies inside).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

__all__ = ["lib", "fmha_forward", "fmha_fwd", "fmha_fwd_host", "fmha_fwd_reference", "attention_flops",
           "save_tensor", "load_tensor", "FmhaError", "LIB_PATH", "CLI_PATH", "F16", "BF16"]

HERE = os.path.dirname(os.path.abspath(__file__))
# FMHA_B200_LIB selects an alternative build (e.g. build/libfmha_b200_trace.so)
LIB_PATH = os.environ.get("FMHA_B200_LIB") or os.path.join(HERE, "libfmha_b200.so")

F16 = 0
BF16 = 1
OK, ERR_CONFIG, ERR_CUDA, ERR_UNSUPPORTED = 0, 2, 5, 6


class FmhaError(RuntimeError):
    """A CUDA-side failure of the FMHA library (status FMHA_ERR_CUDA)."""


class FwdParams(C.Structure):
    """fmha_fwd_params (include/fmha/fmha.h)."""
    _fields_ = [("L", C.c_int64), ("N", C.c_int64), ("h", C.c_int64), ("d", C.c_int64),
                ("q_stride", C.c_int64 * 3), ("k_stride", C.c_int64 * 3),
                ("v_stride", C.c_int64 * 3), ("o_stride", C.c_int64 * 3),
                ("scale", C.c_float), ("dtype", C.c_int)]


_lib = None


def lib():
    """Load the sm_100a library (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: build it with `make` or __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER(FwdParams)
        vp = C.c_void_p
        L.fmha_params_dense.argtypes = [P, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_float]
        L.fmha_params_dense.restype = None
        L.fmha_fwd_check.argtypes = [P]
        L.fmha_fwd_check.restype = C.c_int
        L.fmha_fwd.argtypes = [P, vp, vp, vp, vp, vp, vp]
        L.fmha_fwd.restype = C.c_int
        L.fmha_fwd_host.argtypes = [P, vp, vp, vp, vp, vp, C.c_int]
        L.fmha_fwd_host.restype = C.c_int
        L.fmha_forward_f32.argtypes = [vp, vp, vp] + [C.c_int64] * 6 + [C.c_int, C.c_float, vp, vp, C.c_int]
        L.fmha_forward_f32.restype = C.c_int
        L.fmha_attention_flops.argtypes = [C.c_int64] * 4
        L.fmha_attention_flops.restype = C.c_int64
        L.fmha_last_error.restype = C.c_char_p
        L.fmha_last_launch_count.restype = C.c_int
        L.fmha_kernel_for.argtypes = [P]
        L.fmha_kernel_for.restype = C.c_char_p
        L.fmha_version.restype = C.c_char_p
        L.fmha_host_quantize.argtypes = [vp, vp, C.c_int64, C.c_int]
        L.fmha_host_quantize.restype = None
        L.fmha_host_dequantize.argtypes = [vp, vp, C.c_int64, C.c_int]
        L.fmha_host_dequantize.restype = None
        L.fmha_host_f32_to_16.argtypes = [C.c_float, C.c_int]
        L.fmha_host_f32_to_16.restype = C.c_uint16
        L.fmha_host_16_to_f32.argtypes = [C.c_uint16, C.c_int]
        L.fmha_host_16_to_f32.restype = C.c_float
        L.fmha_tensor_save.argtypes = [C.c_char_p, vp] + [C.c_int64] * 4 + [C.c_int]
        L.fmha_tensor_save.restype = C.c_int
        L.fmha_tensor_load_header.argtypes = [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int)]
        L.fmha_tensor_load_header.restype = C.c_int
        L.fmha_tensor_load.argtypes = [C.c_char_p, vp, C.c_int64]
        L.fmha_tensor_load.restype = C.c_int
        L.fmha_fwd_reference.argtypes = [P, vp, vp, vp, vp, vp, vp]
        L.fmha_fwd_reference.restype = C.c_int
        _lib = L
    return _lib


def _raise(status: int):
    msg = lib().fmha_last_error().decode()
    if status in (ERR_CONFIG, ERR_UNSUPPORTED):
        raise ValueError(msg)
    raise FmhaError(f"fmha status {status}: {msg}")


def _dtype_code(precision) -> int:
    p = str(precision).lower().replace("torch.", "")
    if p in ("f16", "f16emu", "fp16", "float16", "half"):
        return F16
    if p in ("bf16", "bfloat16"):
        return BF16
    if p in ("f32", "exactf32", "float32"):
        raise ValueError("the GPU path is 16-bit: precision must be 'f16emu'/'f16' or 'bf16'")
    raise ValueError("precision must be 'f16emu', 'f16' or 'bf16'")


def attention_flops(L, N, h, d) -> int:
    """4 * N^2 * d * h * L (attention_flops, attention.cpp:191-193)."""
    return int(lib().fmha_attention_flops(L, N, h, d))


def dense_params(L, N, h, d, dtype=F16, scale=0.0) -> FwdParams:
    p = FwdParams()
    lib().fmha_params_dense(C.byref(p), L, N, h, d, dtype, float(scale))
    return p


class _OutputPool:
    """Recycled float32 output buffers for :func:`fmha_forward`.

    A fresh 134 MB O array (config 3) costs ~4 ms of first-touch page faults
    inside the call's dequantisation -- a third of the whole reference-shape
    call (tools/exp/f32_path.py).  Buffers are plain bytearrays kept here; one
    is handed out again only when no array or view refers to it any more (its
    reference count is back to the pool's own), so a caller never sees two
    live results share memory."""

    def __init__(self, max_bytes=8 << 30):
        self.bufs: list[bytearray] = []
        self.max_bytes = max_bytes

    def get(self, shape):
        import sys
        nbytes = int(np.prod(shape)) * 4
        buf = None
        for b in self.bufs:
            # references: self.bufs, the loop variable, getrefcount's argument
            if len(b) == nbytes and sys.getrefcount(b) <= 3:
                buf = b
                break
        if buf is None:
            if sum(len(b) for b in self.bufs) + nbytes > self.max_bytes:
                self.bufs = [b for b in self.bufs if sys.getrefcount(b) > 3]
            buf = bytearray(nbytes)
            if nbytes >= (1 << 20):
                self.bufs.append(buf)
        return np.frombuffer(buf, dtype=np.float32).reshape(shape)


_out_pool = _OutputPool()


def fmha_forward(q, k, v, bM=64, bN=64, precision="f16emu", scale=None, return_lse=False, device=0):
    """Reference call shape (bindings.cpp:81-91) on the GPU.

    q, k, v: float32 arrays (L, N, h, d).  Inputs are rounded RNE to the
    16-bit type (fp16 saturating like the reference's f16_round).  Returns
    float32 O (and LSE (L, h, N) when ``return_lse``)."""
    dt = _dtype_code(precision)
    arrs = [np.ascontiguousarray(x, dtype=np.float32) for x in (q, k, v)]
    for a in arrs:
        if a.ndim != 4:
            raise ValueError("expected a (L,N,h,d) array")
    if not (arrs[0].shape == arrs[1].shape == arrs[2].shape):
        raise ValueError("AttentionProblem: Q/K/V shape mismatch")
    L, N, h, d = arrs[0].shape
    o = _out_pool.get((L, N, h, d))
    lse = _out_pool.get((L, h, N)) if return_lse else None
    st = lib().fmha_forward_f32(arrs[0].ctypes.data, arrs[1].ctypes.data, arrs[2].ctypes.data,
                                L, N, h, d, bM, bN, dt, float(scale or 0.0), o.ctypes.data,
                                lse.ctypes.data if lse is not None else None, device)
    if st:
        _raise(st)
    return (o, lse) if return_lse else o


def _strides(t, name):
    s = t.stride()
    if s[3] != 1:
        raise ValueError(f"{name}: head-dim stride must be 1")
    return (C.c_int64 * 3)(s[0], s[1], s[2])


_params_cache: dict = {}


def _fwd_params(q, k, v, o, scale):
    """FwdParams for this call, cached by (shape, strides, dtype, scale): small
    problems are bound by the host-side cost of the call itself."""
    key = (tuple(q.shape), q.stride(), k.stride(), v.stride(), o.stride(), q.dtype, scale)
    p = _params_cache.get(key)
    if p is None:
        import torch
        L, N, h, d = q.shape
        p = FwdParams()
        p.L, p.N, p.h, p.d = L, N, h, d
        p.q_stride, p.k_stride, p.v_stride, p.o_stride = (_strides(q, "q"), _strides(k, "k"),
                                                          _strides(v, "v"), _strides(o, "o"))
        p.scale = float(scale or 0.0)
        p.dtype = BF16 if q.dtype == torch.bfloat16 else F16
        if len(_params_cache) > 256:
            _params_cache.clear()
        _params_cache[key] = p
    return p


def fmha_fwd(q, k, v, o=None, lse=None, scale=None, stream=None, want_lse=True):
    """Device entry point on torch CUDA tensors (L, N, h, d) fp16/bf16.

    Returns (o, lse); allocates o / lse when not given.  Runs on ``stream``
    (a torch.cuda.Stream) or the current stream of q's device."""
    import torch

    if q.dtype not in (torch.float16, torch.bfloat16):
        raise ValueError("q/k/v must be float16 or bfloat16")
    if not (q.dtype == k.dtype == v.dtype):
        raise ValueError("q/k/v dtypes differ")
    if not (q.shape == k.shape == v.shape) or q.dim() != 4:
        raise ValueError("AttentionProblem: Q/K/V shape mismatch")
    dev = q.device
    if dev.type != "cuda" or k.device != dev or v.device != dev:
        raise ValueError("q/k/v must be CUDA tensors on one device")
    L, N, h, d = q.shape
    if o is None:
        o = torch.empty_like(q, memory_format=torch.contiguous_format)
    elif o.shape != q.shape or o.dtype != q.dtype or o.device != dev:
        raise ValueError(f"o must be a {q.dtype} tensor of shape {tuple(q.shape)} on {dev}")
    if lse is None and want_lse:
        lse = torch.empty((L, h, N), dtype=torch.float32, device=dev)
    elif lse is not None and (lse.shape != (L, h, N) or lse.dtype != torch.float32 or lse.device != dev
                              or not lse.is_contiguous()):
        raise ValueError(f"lse must be a contiguous float32 tensor of shape {(L, h, N)} on {dev}")
    p = _fwd_params(q, k, v, o, scale)
    args = (C.byref(p), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
            lse.data_ptr() if lse is not None else None)
    if dev.index == torch.cuda.current_device():
        st = lib().fmha_fwd(*args, (stream or torch.cuda.current_stream(dev)).cuda_stream)
    else:  # launch on q's device (the ABI uses the current one)
        with torch.cuda.device(dev):
            st = lib().fmha_fwd(*args, (stream or torch.cuda.current_stream(dev)).cuda_stream)
    if st:
        _raise(st)
    return o, lse


def fmha_fwd_host(q, k, v, o, lse=None, dtype=F16, scale=None, device=0):
    """Host 16-bit buffers (numpy uint16 / float16 arrays, (L, N, h, d), dense):
    H2D copies, kernel, D2H copies, synchronise.  Writes o (and lse)."""
    L, N, h, d = q.shape
    p = dense_params(L, N, h, d, dtype, scale or 0.0)
    for a in (q, k, v, o):
        if not a.flags["C_CONTIGUOUS"] or a.itemsize != 2:
            raise ValueError("host buffers must be dense 16-bit arrays")
    st = lib().fmha_fwd_host(C.byref(p), q.ctypes.data, k.ctypes.data, v.ctypes.data, o.ctypes.data,
                             lse.ctypes.data if lse is not None else None, device)
    if st:
        _raise(st)
    return o, lse


def save_tensor(t, path, precision="f32"):
    """FHMT fixture file (the reference's save_tensor, tensor.cpp:30-60)."""
    if precision not in ("f32", "f16"):
        raise ValueError("save_tensor: unknown precision " + str(precision))
    t = np.ascontiguousarray(t, np.float32)
    if t.ndim != 4:
        raise ValueError("expected a (L,N,h,d) array")
    L, N, h, d = t.shape
    st = lib().fmha_tensor_save(str(path).encode(), t.ctypes.data, L, N, h, d, int(precision == "f16"))
    if st:
        raise RuntimeError(lib().fmha_last_error().decode())


def load_tensor(path):
    """Read an FHMT fixture file (the reference's load_tensor, tensor.cpp:62-84)."""
    dims = (C.c_int64 * 4)()
    f16 = C.c_int(0)
    if lib().fmha_tensor_load_header(str(path).encode(), dims, C.byref(f16)):
        raise RuntimeError(lib().fmha_last_error().decode())
    out = np.empty(tuple(int(x) for x in dims), np.float32)
    if lib().fmha_tensor_load(str(path).encode(), out.ctypes.data, out.size):
        raise RuntimeError(lib().fmha_last_error().decode())
    return out


def fmha_fwd_reference(q, k, v, scale=None):
    """Verification path: the fp32 CUDA-core standard attention
    (attention.cpp:137-151 semantics) on torch CUDA 16-bit tensors.
    Returns fp32 (O (L, N, h, d), LSE (L, h, N))."""
    import torch
    L, N, h, d = q.shape
    p = FwdParams()
    p.L, p.N, p.h, p.d = L, N, h, d
    p.q_stride, p.k_stride, p.v_stride, p.o_stride = (_strides(q, "q"), _strides(k, "k"),
                                                      _strides(v, "v"), (C.c_int64 * 3)(N * h * d, h * d, d))
    p.scale = float(scale or 0.0)
    p.dtype = BF16 if q.dtype == torch.bfloat16 else F16
    o = torch.empty((L, N, h, d), dtype=torch.float32, device=q.device)
    lse = torch.empty((L, h, N), dtype=torch.float32, device=q.device)
    st = lib().fmha_fwd_reference(C.byref(p), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                  lse.data_ptr(), torch.cuda.current_stream(q.device).cuda_stream)
    if st:
        _raise(st)
    return o, lse


CLI_PATH = os.path.join(HERE, "fmha-b200")


def kernel_for(L, N, h, d, dtype=F16) -> str:
    """Name of the kernel fmha_fwd launches for a dense (L, N, h, d) problem
    (host-only query of the dispatcher)."""
    p = dense_params(L, N, h, d, _dtype_code(dtype) if isinstance(dtype, str) else dtype)
    name = lib().fmha_kernel_for(C.byref(p))
    if name is None:
        _raise(lib().fmha_fwd_check(C.byref(p)))
    return name.decode()


def launch_count() -> int:
    """Kernel launches issued by the last fmha_fwd call on this thread."""
    return int(lib().fmha_last_launch_count())
