"""bench.py keeps the driver's JSON-line contract (run tiny on the GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline",
        "clocks"]


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_line_has_contract_keys():
    d = _run("--steps", "2", "--warmup", "3", "--sim-steps", "200", "--no-cpu-baseline")
    for k in KEYS:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] >= 3
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["gpu_launches"] == 2
    r = d["roofline"]
    assert 0 < r["frac"] < 1 and r["peak"] > 0 and abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
    # the stream's own ceiling sits below the lookup peak
    assert 0 < r["rng_ceiling_frac"] < 1 and 0 < r["frac_of_rng_ceiling"] < 1
    assert d["config"]["workload"].startswith("c2")


@pytest.mark.gpu
def test_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["e2e"]["h2d_bytes_per_step"] == 0


def test_gpus_flag_launches_one_rank_per_gpu(monkeypatch):
    """`bench.py --gpus N` outside torchrun re-launches itself as N ranks
    through torch.distributed.run on 127.0.0.1 (the driver's own launch);
    under torchrun, WORLD_SIZE must match --gpus."""
    sys.path.insert(0, ROOT)
    import bench

    seen = {}
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    a = bench.parse()
    with pytest.raises(SystemExit):
        bench.launch_ranks(a)
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-3:] == ["--gpus", "4", "--steps", "2"][-3:]
    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit):
        bench.launch_ranks(a)  # WORLD_SIZE 2 != --gpus 4
    monkeypatch.setenv("WORLD_SIZE", "4")
    assert bench.launch_ranks(a) is False
    monkeypatch.delenv("WORLD_SIZE")
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    assert bench.launch_ranks(bench.parse()) is False  # N = 1: no re-launch
