"""`fmha-b200` -- the GPU counterpart of the reference CLI `fmha-sim`
(proj/tools/fmha_cli.cpp): flags, exit codes (0 ok / 2 config / 3 verify,
fmha_cli.cpp:19-22; 5 CUDA), verify against the fp32 device checker, FHMT
dump/load, and the sweep over the paper's shapes."""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_2312_11918_b200 as fm


def run(*args, timeout=600):
    assert os.path.exists(fm.CLI_PATH), "build the CLI with make"
    return subprocess.run([fm.CLI_PATH, *map(str, args)], capture_output=True, text=True, timeout=timeout)


@pytest.mark.parametrize("args,msg", [
    (("verify", "--seqlen", 100, "--tile-q", 64), "must be divisible"),  # validate_tiling
    (("verify", "--seqlen", 96, "--tile-k", 64), "must be divisible"),
    (("verify", "--headdim", 32), "unsupported"),
    (("verify", "--precision", "f32"), "16-bit"),
    (("verify", "--format", "xml"), "--format"),
    (("verify", "--bogus"), "unknown flag"),
    (("frobnicate",), "unknown subcommand"),
    (("verify", "--seqlen"), "needs a value"),
])
def test_config_errors_exit_2(args, msg):
    """cli_integration.cmake:55-58: bad tiling / bad flags exit 2 before any GPU work."""
    r = run(*args)
    assert r.returncode == 2, r.stderr
    assert msg in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("d,prec", [(64, "f16emu"), (128, "bf16"), (256, "f16emu")])
def test_verify_passes(d, prec):
    r = run("verify", "--seqlen", 512, "--headdim", d, "--heads", 2, "--batch", 2, "--precision", prec,
            "--format", "json", "--iterations", 3)
    assert r.returncode == 0, r.stdout + r.stderr
    j = json.loads(r.stdout)
    assert j["pass"] and j["max_abs_error"] <= 1e-2 and j["lse_rel_error"] <= 1e-4
    assert j["tflops"] > 0


@pytest.mark.gpu
def test_verify_text_and_dump_load_round_trip(tmp_path, oracle):
    prefix = str(tmp_path / "c1")
    r = run("verify", "--seqlen", 512, "--headdim", 64, "--heads", 1, "--dump-prefix", prefix)
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout + r.stderr
    q = fm.load_tensor(prefix + "_q.fhmt")
    # the CLI's generator reproduces the reference fixtures (seed 42, random.hpp)
    np.testing.assert_array_equal(q, oracle.quantize(oracle.gaussian(1, 512, 1, 64, 42), "f16"))
    o = fm.load_tensor(prefix + "_o.fhmt")
    qq, kk, vv = oracle.problem(1, 512, 1, 64, 42, dtype="f16")
    o_ref, _ = oracle.fmha_forward(qq, kk, vv, 128, 128)
    assert np.abs(o - o_ref).max() < 1e-2
    r2 = run("verify", "--load-prefix", prefix, "--format", "csv")
    assert r2.returncode == 0, r2.stderr
    assert r2.stdout.splitlines()[0].startswith("config,ms,tflops")


@pytest.mark.gpu
def test_sweep_reports_paper_shapes():
    r = run("sweep", "--format", "json", "--iterations", 5)
    assert r.returncode == 0, r.stderr
    rows = json.loads(r.stdout)
    assert [x["config"] for x in rows] == ["L=4,N=4096,h=32,d=64,fp16", "L=4,N=4096,h=16,d=128,fp16",
                                           "L=4,N=4096,h=8,d=256,fp16"]
    assert all(x["tflops"] > 100 for x in rows)


@pytest.mark.gpu
@pytest.mark.parametrize("d", [64, 128, 256])
def test_device_checker_matches_oracle(oracle, d):
    """The CLI's checker (fp32 CUDA-core standard attention) against the CPU oracle."""
    import torch
    q, k, v = oracle.problem(2, 200, 3, d, 31, dtype="bf16")
    tq, tk, tv = (torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (q, k, v))
    o, lse = fm.fmha_fwd_reference(tq, tk, tv)
    torch.cuda.synchronize()
    o_ref, lse_ref = oracle.standard_attention(q, k, v)
    assert np.abs(o.cpu().numpy() - o_ref).max() < 2e-5
    assert np.abs((lse.cpu().numpy() - lse_ref) / lse_ref).max() < 1e-5
