"""Where the reference-call-shape path (fmha_forward_f32) spends its time, c3."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2312_11918_b200 as fm
import ctypes as C
L, N, h, d = 4, 4096, 16, 128
rng = np.random.default_rng(0)
q, k, v = (rng.standard_normal((L, N, h, d), dtype=np.float32) for _ in range(3))
for _ in range(2):
    fm.fmha_forward(q, k, v, 128, 128, return_lse=True)
t = time.perf_counter(); n = 5
for _ in range(n):
    fm.fmha_forward(q, k, v, 128, 128, return_lse=True)
print(f"fmha_forward (fresh output arrays): {(time.perf_counter() - t) / n * 1e3:.2f} ms")
o = np.empty_like(q); lse = np.empty((L, h, N), np.float32)
o.fill(0); lse.fill(0)
lib = fm.lib()
t = time.perf_counter()
for _ in range(n):
    st = lib.fmha_forward_f32(q.ctypes.data, k.ctypes.data, v.ctypes.data, L, N, h, d, 128, 128, 0, 0.0,
                              o.ctypes.data, lse.ctypes.data, 0)
print(f"fmha_forward_f32 (preallocated, touched output): {(time.perf_counter() - t) / n * 1e3:.2f} ms")
t = time.perf_counter()
for _ in range(n):
    x = np.empty_like(q); x.fill(0)
print(f"np.empty + fill of a 268 MB... (O-sized 134 MB) array: {(time.perf_counter() - t) / n * 1e3:.2f} ms")
b16 = np.empty(q.size, np.uint16)
t = time.perf_counter()
for _ in range(n):
    for a in (q, k, v):
        lib.fmha_host_quantize(a.ctypes.data, b16.ctypes.data, a.size, 0)
print(f"quantize Q,K,V (402 MB float): {(time.perf_counter() - t) / n * 1e3:.2f} ms")
t = time.perf_counter()
for _ in range(n):
    lib.fmha_host_dequantize(b16.ctypes.data, o.ctypes.data, o.size, 0)
print(f"dequantize O (134 MB float): {(time.perf_counter() - t) / n * 1e3:.2f} ms")
