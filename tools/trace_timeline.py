"""Debug: per-K/V-tile timeline of CTA 0's first work unit (FMHA_TRACE=1),
per-warp completion skew, and the per-unit timeline of CTA 0.

Run on a GPU (needs `make trace`):
    FMHA_TRACE=1 python tools/trace_timeline.py [N] [d] [L] [h]

Slots per (Q tile q, K/V tile j), see FwdArgs::trace in fmha_fwd_kernel.cuh:
 softmax WG q: 0 woke (S ready)  1 S in registers  8 row max done  9 first-half exps
               2 first half published  10 second-half exps  3 second half published
 MMA warp:     4 saw P half 0  11 saw P half 1  12 PV issued  5 S(j+1) issued
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FMHA_B200_LIB", os.path.join(ROOT, "build", "libfmha_b200_trace.so"))
os.environ.setdefault("FMHA_TRACE", "1")
import paper_2312_11918_b200 as fm  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
d = int(sys.argv[2]) if len(sys.argv) > 2 else 128
L = int(sys.argv[3]) if len(sys.argv) > 3 else 4
h = int(sys.argv[4]) if len(sys.argv) > 4 else 16
q, k, v = (torch.randn(L, N, h, d, device="cuda").half() for _ in range(3))
for _ in range(3):
    fm.fmha_fwd(q, k, v)
torch.cuda.synchronize()
S = 16
n_kv = (N + 127) // 128
buf = np.zeros(3 * n_kv * S + 64, np.uint64)
fm.lib().fmha_debug_trace_copy(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), buf.size)
full = buf[:3 * n_kv * S].reshape(-1, n_kv, S).astype(np.int64)
units = buf[3 * n_kv * S: 3 * n_kv * S + 64].reshape(8, 8).astype(np.int64)
t = full[:2]
warp_t = full[2].astype(np.int64)
start, setup = t[0, 0, 6], t[0, 0, 7]
t = np.where(t > 0, t - start, -1)

SEG = [  # (name, from slot, to slot, same j?)
    ("S ready->in regs", 0, 1), ("row max", 1, 8), ("exp half0", 8, 9), ("publish0", 9, 2),
    ("exp half1", 2, 10), ("publish1", 10, 3), ("P1 arrive->MMA saw", 3, 11), ("PV issue", 11, 12),
    ("S issue", 12, 5),
]
print(f"N={N} d={d} n_kv={n_kv}  setup {setup - start} clk, first S ready q0 {t[0,0,0]} q1 {t[1,0,0]}")
lo, hi = min(2, n_kv - 1), max(n_kv - 2, min(2, n_kv - 1) + 1)
for name, a, b in SEG:
    vals = t[:, lo:hi, b] - t[:, lo:hi, a]
    print(f"  {name:22s} median q0 {np.median(vals[0]):6.0f}  q1 {np.median(vals[1]):6.0f}")
issue_to_next = t[:, lo + 1:hi + 1, 0] - t[:, lo:hi, 5]
print(f"  {'S issued->next wake':22s} median q0 {np.median(issue_to_next[0]):6.0f}  q1 {np.median(issue_to_next[1]):6.0f}")
per = np.diff(t[0, lo:hi, 0])
if per.size:
    print(f"steady-state period per K/V tile: median {np.median(per):.0f} clk, min {per.min()}")
# overlap of the two softmax WGs' busy intervals [in regs, published]
busy0 = [(t[0, j, 1], t[0, j, 3]) for j in range(lo, hi)]
busy1 = [(t[1, j, 1], t[1, j, 3]) for j in range(lo, hi)]
ov = 0
for a0, b0 in busy0:
    for a1, b1 in busy1:
        ov += max(0, min(b0, b1) - max(a0, a1))
tot = t[0, hi - 1, 3] - t[0, lo, 1]
print(f"softmax WG busy fraction: q0 {sum(b - a for a, b in busy0) / tot:.2f}  q1 {sum(b - a for a, b in busy1) / tot:.2f}  "
      f"overlapped {ov / tot:.2f}")
print("\nraw timeline, tiles 4..6 (clk since kernel start):")
ev = []
names = {0: "wake", 1: "ld", 8: "max", 9: "exp0", 2: "pub0", 10: "exp1", 3: "pub1", 4: "mma saw P0", 11: "mma saw P1",
         12: "PV issued", 5: "S issued"}
for j in range(4, min(7, n_kv)):
    for qq in range(2):
        for sl, nm in names.items():
            if t[qq, j, sl] >= 0:
                ev.append((t[qq, j, sl], f"q{qq} j{j} {nm}"))
for x, nm in sorted(ev):
    print(f"  {x:8d}  {nm}")
for qq in range(2):
    print(f"q{qq}: last P {t[qq,-1,3]}  O ready {t[qq,-1,6]}  epilogue done {t[qq,-1,7]}  "
          f"mainloop {(t[qq,-1,3]-t[qq,0,0])/n_kv:.0f} clk/tile")


w = warp_t - start
print("\nper-warp P-complete time minus the tile's earliest (warp w: tile w//4, SM sub-partition w%4), tiles 4..9:")
for j in range(4, min(10, n_kv)):
    for qq in range(2):
        ws = [4 * qq + x for x in range(4)]
        base = min(w[j, x] for x in ws)
        print(f"  j{j} q{qq}: " + " ".join(f"w{x}:{w[j, x] - base:5d}" for x in ws))

print("\nper-unit timeline of CTA 0 (clk since kernel start): Q ready at MMA | first S ready q0 q1 | epilogue done q0 q1")
for i in range(8):
    if units[i, 0] == 0:
        break
    x = [v - start if v > 0 else -1 for v in units[i, :5]]
    print(f"  unit {i}: {x[0]:8d} | {x[1]:8d} {x[2]:8d} | {x[3]:8d} {x[4]:8d}")
