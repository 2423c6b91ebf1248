"""Debug: print the per-iteration timeline of CTA (0,0,0) (FMHA_TRACE=1).
Run on a GPU:  FMHA_TRACE=1 python tools/trace_timeline.py [N] [d]"""
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
L, h = 4, 16
q, k, v = (torch.randn(L, N, h, d, device="cuda").half() for _ in range(3))
for _ in range(3):
    fm.fmha_fwd(q, k, v)
torch.cuda.synchronize()
n_kv = (N + 127) // 128
buf = np.zeros(2 * n_kv * 8, np.uint64)
fm.lib().fmha_debug_trace_copy(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), buf.size)
t = buf.reshape(2, n_kv, 8).astype(np.int64)
t0 = t[0, 0, 6]
t = np.where(t > 0, t - t0, -1)
names = ["wake", "ld", "max", "P+arrive", "mma_sawP", "mma_issued"]
print("q j | " + " ".join(f"{n:>10s}" for n in names) + " | ld  max  exp  P->mma  issue")
for j in range(min(n_kv, 12)):
    for qq in range(2):
        r = t[qq, j]
        print(f"{qq} {j:2d} | " + " ".join(f"{x:10d}" for x in r[:6]) +
              f" | {r[1]-r[0]:4d} {r[2]-r[1]:4d} {r[3]-r[2]:5d} {r[4]-r[3]:6d} {r[5]-r[4]:5d}")
if n_kv > 3:
    per = np.diff(t[0, 2:n_kv - 1, 0])
    print("steady-state period per K/V tile (clk): median", int(np.median(per)), "min", int(per.min()))
if n_kv <= 3:
    sys.exit(0)
d_ld = np.median(t[:, 2:-1, 1] - t[:, 2:-1, 0]); d_max = np.median(t[:, 2:-1, 2] - t[:, 2:-1, 1])
d_exp = np.median(t[:, 2:-1, 3] - t[:, 2:-1, 2]); d_p2m = np.median(t[:, 2:-2, 4] - t[:, 2:-2, 3])
d_iss = np.median(t[:, 2:-2, 5] - t[:, 2:-2, 4])
d_tc = np.median(t[:, 3:-1, 0] - t[:, 2:-2, 5])
print(f"median: ldtm {d_ld:.0f}  max {d_max:.0f}  exp+store+arrive {d_exp:.0f}  P->MMA wake {d_p2m:.0f}  "
      f"MMA issue {d_iss:.0f}  issue->S ready {d_tc:.0f}")

print(f"kernel start -> setup done {t[0,0,7]}  first S ready (q0) {t[0,0,0]}  (q1) {t[1,0,0]}")
for qq in range(2):
    print(f"q{qq}: last P arrive {t[qq,-1,3]}  O ready {t[qq,-1,6]}  epilogue done {t[qq,-1,7]}  "
          f"(mainloop {t[qq,-1,3]-t[qq,0,0]} clk for {n_kv} tiles = {(t[qq,-1,3]-t[qq,0,0])/n_kv:.0f}/tile)")
