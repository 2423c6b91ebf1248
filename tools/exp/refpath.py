import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2312_11918_b200 as fm
rng = np.random.default_rng(0)
L, N, h, d = 4, 4096, 16, 128
q, k, v = (rng.standard_normal((L, N, h, d), dtype=np.float32) for _ in range(3))
for _ in range(2):
    fm.fmha_forward(q, k, v, 64, 64, "f16emu")
ts = []
for _ in range(5):
    t0 = time.perf_counter(); o = fm.fmha_forward(q, k, v, 64, 64, "f16emu"); ts.append(time.perf_counter() - t0)
fl = 4 * L * N * N * h * d
print(f"fmha_forward (reference call shape, float32 host arrays, c3): best {min(ts)*1e3:.1f} ms, median {sorted(ts)[2]*1e3:.1f} ms -> {fl/min(ts)/1e12:.1f} TFLOP/s")
