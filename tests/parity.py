"""Shared helpers for the GPU parity tests (test infrastructure).

The oracle is the C restatement of the reference (oracle/fmha_oracle.c),
pinned bit-exactly to the reference build (tests/test_oracle.py).  The
tolerances are BASELINE.json's north-star ones:
  O: max abs err <= 1e-2, mean abs err <= 1e-3;  LSE: rel err <= 1e-4.
"""
import numpy as np

O_MAX_ABS = 1e-2
O_MEAN_ABS = 1e-3
LSE_REL = 1e-4


def torch_dtype(dt):
    import torch
    return torch.bfloat16 if dt == "bf16" else torch.float16


def gpu_fmha(q, k, v, dt, scale=None, device="cuda:0", want_lse=True):
    """Run the B200 kernel on float32 inputs that are already exactly
    representable in `dt`.  Returns float32 numpy (O, LSE)."""
    import torch
    import paper_2312_11918_b200 as fm
    tq, tk, tv = (torch.from_numpy(np.ascontiguousarray(x)).to(device).to(torch_dtype(dt)) for x in (q, k, v))
    o, lse = fm.fmha_fwd(tq, tk, tv, scale=scale, want_lse=want_lse)
    torch.cuda.synchronize()
    return o.float().cpu().numpy(), (lse.cpu().numpy() if lse is not None else None)


def errors(o, lse, o_ref, lse_ref):
    diff = np.abs(o.astype(np.float64) - o_ref.astype(np.float64))
    res = {"max_abs": float(diff.max()), "mean_abs": float(diff.mean()),
           # the reference's own metric, |a-b| / max(|b|, 1) (fmha_cli.cpp:63-77)
           "max_rel_ref": float((diff / np.maximum(np.abs(o_ref), 1.0)).max())}
    if lse is not None and lse_ref is not None:
        res["lse_rel"] = float((np.abs(lse.astype(np.float64) - lse_ref) / np.abs(lse_ref)).max())
    return res


def assert_within(res, ctx=""):
    assert np.isfinite(res["max_abs"]), f"non-finite output {ctx}"
    assert res["max_abs"] <= O_MAX_ABS, f"O max abs {res['max_abs']:.3e} > {O_MAX_ABS} {ctx}"
    assert res["mean_abs"] <= O_MEAN_ABS, f"O mean abs {res['mean_abs']:.3e} > {O_MEAN_ABS} {ctx}"
    if "lse_rel" in res:
        assert res["lse_rel"] <= LSE_REL, f"LSE rel {res['lse_rel']:.3e} > {LSE_REL} {ctx}"
