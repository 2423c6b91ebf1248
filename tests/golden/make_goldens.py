"""Generate tests/golden/* from the REFERENCE itself (oracle/_ref, compiled
from /root/reference/proj/src by oracle/Makefile).  Run in the dev container
(where /root/reference exists):  python tests/golden/make_goldens.py

Outputs
  goldens.json   FNV-1a-64 hashes (32-bit-word FNV over float storage order)
                 of reference outputs: SURVEY.md Appendix A values plus the
                 acceptance criterion-3 grid (proj/tests/acceptance.cpp:71-96).
  c1_ref.npz     reference O and LSE for config 1 (L=1,h=1,N=512,d=64,
                 seeds 42/43/44) on inputs pre-rounded to f16 and to bf16,
                 tile 128x128 -- the GPU parity fixture.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as orc  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    if not orc.ref_available():
        orc.build()
    assert orc.ref_available(), "oracle/_ref not built (needs /root/reference)"
    g = {}
    q, k, v = (orc.ref_gaussian(1, 512, 1, 64, s) for s in (42, 43, 44))
    g["gaussian_1_512_1_64"] = {str(s): orc.fnv1a64(t) for s, t in zip((42, 43, 44), (q, k, v))}
    g["gaussian_first3_seed42"] = [float(x) for x in q.reshape(-1)[:3]]
    g["c1_fmha"] = {}
    for bm in (64, 128):
        for prec, name in ((0, "f32"), (1, "f16emu")):
            o = orc.ref_fmha_forward(q, k, v, bm, bm, prec)
            g["c1_fmha"][f"{bm}x{bm}_{name}"] = orc.fnv1a64(o)
            if bm == 64:
                g[f"c1_first3_{name}"] = [float(x) for x in o.reshape(-1)[:3]]
    g["c1_standard_f32"] = orc.fnv1a64(orc.ref_standard_attention(q, k, v))
    qq, kk, vv = (orc.quantize(t, "f16") for t in (q, k, v))
    g["c1_f16inputs_64x64_f32"] = orc.fnv1a64(orc.ref_fmha_forward(qq, kk, vv, 64, 64))
    # acceptance criterion 3 grid (seeds 1000 + 10 per (N, d) pair)
    grid = {}
    seed = 1000
    for N in (128, 256, 512):
        for d in (64, 128, 256):
            a, b, c = (orc.ref_gaussian(1, N, 1, d, seed + i) for i in range(3))
            for bm in (64, 128):
                for bn in (64, 128):
                    grid[f"N{N}_d{d}_{bm}x{bn}_seed{seed}"] = orc.fnv1a64(orc.ref_fmha_forward(a, b, c, bm, bn))
            seed += 10
    g["acceptance_c3_grid"] = grid
    with open(os.path.join(OUT, "goldens.json"), "w") as f:
        json.dump(g, f, indent=1, sort_keys=True)

    fx = {}
    for dt in ("f16", "bf16"):
        a, b, c = (orc.quantize(t, dt) for t in (q, k, v))
        tiles = [(0, 0, i) for i in range(512 // 128)]
        O, lse = orc.ref_fmha_tiles(a, b, c, tiles, 128, 128)
        fx[f"O_{dt}"] = O.reshape(512, 64)
        fx[f"lse_{dt}"] = lse.reshape(512)
    np.savez_compressed(os.path.join(OUT, "c1_ref.npz"), **fx)
    print("wrote goldens.json and c1_ref.npz")


if __name__ == "__main__":
    main()
