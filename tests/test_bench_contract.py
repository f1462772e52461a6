"""bench.py's JSON-line contract, checked on CPU through the reference arm (the fp64 oracle timed
on the host cores; the only leg of bench.py that runs without a GPU), and its host helpers."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.mark.parametrize("cfg", ["tiny", "dec1"])
def test_reference_arm_json_line(cfg):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", cfg,
                          "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "TFLOP/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith(cfg)


def test_warmup_floor_enforced():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "tiny",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode != 0 and "warmup" in (out.stdout + out.stderr)


def test_route_launch_count_rule():
    import bench
    assert bench.route_launches(1, 8, 2) == 1            # single-block small-batch kernel
    assert bench.route_launches(1024, 16, 8) == 1
    assert bench.route_launches(1025, 8, 2) == 2         # histogram + fused placement
    assert bench.route_launches(4096, 8, 2) == 2
    assert bench.route_launches(20000, 1024, 3) == 3     # + the single-block scan


def test_oracle_sample_fp8_bounded():
    import bench
    import synth
    f, s, sample, cores = bench.oracle_sample(synth.CONFIGS["tiny"], 0, 0.01, fp8=True)
    assert f > 0 and s > 0 and "E4M3" in sample and cores >= 1
