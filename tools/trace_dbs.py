"""Debug: per-K/V-step timeline of CTA 0 in the double-buffered-S d=128 kernel
(FMHA_TRACE=1, `make trace`).  Slots: see dbs_stamp in fmha_fwd_dbs_kernel.cuh.
    FMHA_TUNE_DBS=1 python tools/trace_dbs.py [N] [L] [h]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FMHA_B200_LIB", os.path.join(ROOT, "build", "libfmha_b200_trace.so"))
os.environ.setdefault("FMHA_TRACE", "1")
os.environ.setdefault("FMHA_TUNE_DBS", "1")
import paper_2312_11918_b200 as fm  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
h = int(sys.argv[3]) if len(sys.argv) > 3 else 16
q, k, v = (torch.randn(L, N, h, 128, device="cuda").half() for _ in range(3))
for _ in range(3):
    fm.fmha_fwd(q, k, v)
torch.cuda.synchronize()
G = 64
buf = np.zeros(G * 48, np.uint64)
fm.lib().fmha_debug_trace_copy(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), buf.size)
t = buf[:G * 16].reshape(G, 16).astype(np.int64)
wt = buf[G * 16:].reshape(G, 8, 4).astype(np.int64)
t0 = t[0, 0]
wt = np.where(wt > 0, wt - t0, -1)
t = np.where(t > 0, t - t0, -1)
names = ["S seen", "in regs", "max", "h0 exps", "P0 pub", "P1 pub", "w4 S seen", "w4 P1", "V rdy", "MMA P0",
         "MMA P1", "PV iss", "K+2 rdy", "S+2 iss"]
print("step " + " ".join(f"{n:>9s}" for n in names))
for g in range(min(G, 40)):
    print(f"{g:4d} " + " ".join(f"{t[g, k]:9d}" for k in range(14)))
# steady-state averages (steps 8..G-8 of the first unit span)
a, b = 8, min(G, 40) - 2
d = lambda x, y: np.mean([t[g, y] - t[g, x] for g in range(a, b)])
print(f"\nsteady state, steps {a}..{b}: period {np.mean(np.diff(t[a:b, 0])):.0f} clk")
for (n, x, y) in [("S seen -> in regs", 0, 1), ("ld -> max/vote", 1, 2), ("max -> h0 exps", 2, 3),
                  ("h0 exps -> P0 pub", 3, 4), ("P0 pub -> P1 pub", 4, 5), ("P1 pub -> MMA saw P1", 5, 10),
                  ("MMA P1 -> PV issued", 10, 11), ("PV issued -> S+2 issued", 11, 13),
                  ("w0 S seen -> w4 S seen", 0, 6), ("w0 P1 -> w4 P1", 5, 7)]:
    print(f"  {n:26s} {d(x, y):8.0f}")
print(f"  S+2 issued -> S+2 seen (softmax)  {np.mean([t[g + 2, 0] - t[g, 13] for g in range(a, b)]):8.0f}")
print(f"  P1 pub(g) -> S seen(g+1)          {np.mean([t[g + 1, 0] - t[g, 5] for g in range(a, b)]):8.0f}")

print("\nper softmax warp (steps %d..%d), times relative to warp 0's S observed:" % (a, b))
print("warp   S seen   max done   P0 pub   P1 pub")
for w in range(8):
    r = [np.mean([wt[g, w, k] - wt[g, 0, 0] for g in range(a, b)]) for k in range(4)]
    print(f"{w:4d} " + " ".join(f"{x:9.0f}" for x in r))
print(f"MMA saw P0 {np.mean([t[g, 9] - wt[g, 0, 0] for g in range(a, b)]):.0f}  P1 {np.mean([t[g, 10] - wt[g, 0, 0] for g in range(a, b)]):.0f}")
print("MMA warp stamps relative to warp 0's S observed (same step g):")
for k, n in [(15, "loop top"), (8, "V(g) ready"), (9, "P0 seen"), (10, "P1 seen"), (11, "PV issued"), (12, "K(g+2) ready"), (13, "S(g+2) issued"), (14, "S(g+2) commits")]:
    print(f"  {n:14s} {np.mean([t[g, k] - wt[g, 0, 0] for g in range(a, b)]):8.0f}")
print(f"  S(g+2) seen by warp 0: {np.mean([wt[g + 2, 0, 0] - wt[g, 0, 0] for g in range(a, b)]):8.0f}")
