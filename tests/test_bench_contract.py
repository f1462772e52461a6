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


def test_gpus_flag_self_launches_one_rank_per_gpu(monkeypatch):
    """`bench.py --gpus N` without torchrun re-launches itself as N ranks (torch.distributed.run, one
    process per GPU, rendezvous on 127.0.0.1) and returns their exit code (--gpus was a label)."""
    import bench
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2", "--warmup", "3"])
    monkeypatch.setattr("subprocess.call", lambda cmd: calls.append(cmd) or 0)
    with pytest.raises(SystemExit) as ex:
        bench.main()
    assert ex.value.code == 0 and len(calls) == 1
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-6:] == ["--gpus", "4", "--steps", "2", "--warmup", "3"] and cmd[-7].endswith("bench.py")


def test_gpus_flag_must_match_world_size(monkeypatch):
    import bench
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4"])
    with pytest.raises(SystemExit) as ex:
        bench.main()
    assert "WORLD_SIZE=2" in str(ex.value.code)


def test_ep_config_same_for_both_arms():
    """At N > 1 the reference arm prints the config our arm prints (the driver compares them)."""
    import argparse

    import bench
    import synth
    args = argparse.Namespace(bm=0, bn=0, out_dtype="bf16", seed=0, dtype="bf16", ep=False, gpus=8)
    c = bench.ref_config(synth.CONFIGS["mix"], args, 8)
    assert c == bench.ep_config(synth.CONFIGS["mix"], 8, args)
    assert c["workload"].startswith("mix-ep8: E=8 top-2 T=32768 (4096/rank)") and c["parallelism"] == "ep8"
    s = bench.ep_config(synth.CONFIGS["ep"], 8, args)
    assert "T=32768 (4096/rank)" in s["workload"]                        # 8x22B: strong scaling, total T fixed
