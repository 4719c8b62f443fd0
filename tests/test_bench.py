"""bench.py contract: the reference arm (oracle on the host; CPU) and the
b200 arm on a small class (GPU): one JSON line with the contract's keys."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e")


def _run(args, env=None):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    return [json.loads(l) for l in lines]


def test_reference_arm_line():
    out = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-sample", "20000"])
    assert len(out) == 1
    d = out[0]
    assert d["impl"] == "reference"
    for k in KEYS:
        assert k in d, k
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["host"]["nproc"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("GTC-P class A:")


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--ref-sample", "1000"], env)
    assert out == []


@pytest.mark.gpu
def test_b200_arm_line_small_class():
    out = _run(["--size", "T", "--steps", "2", "--warmup", "3", "--no-cpu", "--e2e-steps", "1"])
    assert len(out) == 1
    d = out[0]
    for k in KEYS + ("roofline", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] == "hbm" and d["roofline"]["peak"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
