"""compute-sanitizer memcheck over every kernel family (tools/sanitize_smoke.py:
ragged N, fp16/bf16, d = 64/128/256, the d=64 two-CTA kernel, CTA pairs with a
padding tile, the d=128 CTA-pair kernel).  DESIGN.md §10 has the racecheck /
synccheck readings; memcheck must report zero errors."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    for p in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if p and os.path.exists(p):
            return p
    return None


def test_memcheck_clean():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    san = _sanitizer()
    if san is None:
        pytest.skip("compute-sanitizer not installed")
    r = subprocess.run([san, "--tool", "memcheck", "--error-exitcode", "3", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_smoke.py")],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]


def test_memcheck_clean_double_buffered_s_kernel():
    """The opt-in d = 128 double-buffered-S kernel (FMHA_TUNE_DBS=1) under memcheck."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    san = _sanitizer()
    if san is None:
        pytest.skip("compute-sanitizer not installed")
    r = subprocess.run([san, "--tool", "memcheck", "--error-exitcode", "3", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_smoke.py"), "d128"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, FMHA_TUNE_DBS="1"))
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]


def test_memcheck_clean_d128_pair_kernel():
    """The opt-in d = 128 CTA-pair kernel (FMHA_TUNE_PAIR128_N=8192) under memcheck."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    san = _sanitizer()
    if san is None:
        pytest.skip("compute-sanitizer not installed")
    r = subprocess.run([san, "--tool", "memcheck", "--error-exitcode", "3", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_smoke.py"), "pair128"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, FMHA_TUNE_PAIR128_N="8192"))
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
