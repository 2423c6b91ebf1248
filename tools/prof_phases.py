"""Per-phase time of the d<=128 ping-pong kernel's warps (FMHA_PROF_BUILD):
    make prof && FMHA_TRACE=1 python tools/prof_phases.py [L h N d dtype]
Prints, per role, the average clk per K/V tile spent in each phase."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FMHA_B200_LIB", os.path.join(ROOT, "build", "libfmha_b200_prof.so"))
os.environ.setdefault("FMHA_TRACE", "1")
import paper_2312_11918_b200 as fm  # noqa: E402

L, h, N, d = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (4, 16, 4096, 128)))
dt = torch.bfloat16 if len(sys.argv) > 5 and sys.argv[5] == "bf16" else torch.float16
q, k, v = (torch.randn(L, N, h, d, device="cuda", dtype=dt) for _ in range(3))
for _ in range(3):
    fm.fmha_fwd(q, k, v)
torch.cuda.synchronize()
grid = min(148, L * h * ((N + 255) // 256))
buf = np.zeros(grid * 16 * 8, np.uint64)
fm.lib().fmha_debug_trace_copy(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), buf.size)
acc = buf.reshape(grid, 16, 8).astype(np.float64)
units = L * h * ((N + 255) // 256)
tiles_per_cta = units / grid * ((N + 127) // 128)
names_sm = ["wait S", "ld+mask", "max|spec-h0", "h0 (redo)", "st+h1", "publish", "epilogue", "loop"]
names_mma = ["wait kv", "wait P", "wait o_empty", "issue", "wait Q", "wait kv(j<2)", "-", "-"]
sm = acc[:, 0:8].mean(axis=(0, 1)) / tiles_per_cta
sm1 = acc[:, [1, 5]].mean(axis=(0, 1)) / tiles_per_cta
mma = acc[:, 9].mean(axis=0) / tiles_per_cta
print(f"L={L} h={h} N={N} d={d}: {tiles_per_cta:.0f} K/V tiles per CTA")
print("softmax warps (all):   " + "  ".join(f"{n} {x:6.0f}" for n, x in zip(names_sm, sm)) + f"   total {sm.sum():.0f}")
print("softmax warps SMSP1:   " + "  ".join(f"{n} {x:6.0f}" for n, x in zip(names_sm, sm1)) + f"   total {sm1.sum():.0f}")
ld = acc[:, 8].mean(axis=0) / tiles_per_cta
print(f"TMA producer:          wait kv_empty {ld[0]:6.0f}  other {ld[3]:6.0f}")
print("MMA warp:              " + "  ".join(f"{n} {x:6.0f}" for n, x in zip(names_mma[:6], mma[:6])) + f"   total {mma[:6].sum():.0f}")
wg0 = acc[:, 0:4].mean(axis=(0, 1)) / tiles_per_cta
wg1 = acc[:, 4:8].mean(axis=(0, 1)) / tiles_per_cta
print("softmax WG 0:          " + "  ".join(f"{n} {x:6.0f}" for n, x in zip(names_sm, wg0)) + f"   total {wg0.sum():.0f}")
print("softmax WG 1:          " + "  ".join(f"{n} {x:6.0f}" for n, x in zip(names_sm, wg1)) + f"   total {wg1.sum():.0f}")
