"""bench.py's reference arm runs on CPU (the reference compiled from its sources,
else the oracle port) and prints the contract's JSON line; the workload split
for torchrun ranks follows SURVEY.md 8(e)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--ref-seconds", "2", "--config", "c1"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "TFLOP/s"
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["gpu_launches"] == 0
    assert "cpu_model" in line["cpu_baseline"]
    # the same `config` object as the GPU arm prints (the driver compares them)
    cfg, _, _, global_l = bench.workload("c1", 1, 0)
    assert line["config"] == bench.config_dict(cfg, global_l)


def test_reference_arm_rank_nonzero_is_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--config", "c1"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_workload_split():
    cfg, loc, scaling, global_l = bench.workload("c3", 4, 1)
    assert scaling == "weak" and loc["L"] == 4 and global_l == 16   # c3 per rank, weak scaling
    cfg, loc, scaling, global_l = bench.workload("c5", 8, 3)
    assert scaling == "strong" and loc["L"] == 1 and global_l == 8  # config 5 sharded by batch
    with pytest.raises(SystemExit):
        bench.workload("c5", 3, 0)
    assert bench.flops(4, 4096, 16, 128) == 549755813888
