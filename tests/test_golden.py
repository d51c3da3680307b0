"""Committed golden vectors produced by the unmodified reference
(tests/golden/make_golden.py): the product's model generator and host plan
reproduce them bit-for-bit (CPU), the oracle restatement reproduces the
reference trajectories (CPU), and the CUDA path reproduces them (GPU)."""
import hashlib
import json
import os

import numpy as np
import pytest

from helpers import config_text, plan_digest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MANIFEST = json.load(open(os.path.join(HERE, "manifest.json")))
NAMES = sorted(MANIFEST)


def _setup(pb, name):
    m = MANIFEST[name]
    text, terms = config_text(m["config"], m.get("p"))
    assert hashlib.sha256(text.encode()).hexdigest() == m["model_sha256"]
    plan = pb.prepare(pb.parse_model(text), m["theta"], m["k_max"], m["mgp"])
    fx = np.load(os.path.join(HERE, f"{name}.npz"))
    return m, plan, fx


@pytest.mark.parametrize("name", NAMES)
def test_plan_digest(pb, name):
    m, plan, _ = _setup(pb, name)
    assert plan.n_kept == m["n_kept"]
    assert plan_digest(plan.flat()) == m["plan_digest"]


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("stream", [0, 1])
def test_oracle_reproduces_reference_trajectories(pb, orc, name, stream):
    m, plan, fx = _setup(pb, name)
    pred = (fx["pred_bits"], fx["pred_vals"])
    st, cnt = orc.simulate(plan.view, m["seed"], m["traj_begin"], m["n_traj"], m["n_steps"],
                           step_begin=m["step_begin"], pred=pred, stream=stream)
    assert np.array_equal(st, fx[f"states_s{stream}"])
    assert np.array_equal(cnt, fx[f"counts_s{stream}"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("stream", [0, 1])
def test_device_reproduces_reference_trajectories(pb, name, stream):
    m, plan, fx = _setup(pb, name)
    pred = (fx["pred_bits"], fx["pred_vals"])
    eng = pb.GpuEnsemble(plan)
    st, cnt = eng.simulate(m["seed"], m["n_traj"], m["n_steps"], traj_begin=m["traj_begin"],
                           step_begin=m["step_begin"], pred=pred, stream=stream)
    assert np.array_equal(st, fx[f"states_s{stream}"])
    assert np.array_equal(cnt, fx[f"counts_s{stream}"])


def _without_warps(kernel):
    # warps per CTA follow the ensemble size; the instantiation is the rest
    return ",".join(p for p in kernel.rstrip(">").split(",") if not p.startswith("warps="))


BENCH_FIXTURES = [n for n in NAMES if MANIFEST[n]["k_max"] == 16 and MANIFEST[n]["mgp"] in (8, 12)]


@pytest.mark.gpu
@pytest.mark.parametrize("name", BENCH_FIXTURES)
@pytest.mark.parametrize("stream", [0, 1])
def test_device_reproduces_reference_on_the_benchmarked_kernel(pb, name, stream):
    """The benchmarked plans, on the very kernel instantiation bench.py runs
    for that workload (its ensemble size): same kernel family, lanes per
    trajectory, gather mode, stream and plan placement."""
    import bench

    m, plan, fx = _setup(pb, name)
    bench_traj = bench.WORKLOADS[m["config"]]["n_traj"]
    want = _without_warps(pb.GpuEnsemble(plan).plan_launch(bench_traj, stream))
    eng = pb.GpuEnsemble(plan, lanes_per_traj=1 if want.startswith("lane") else 0)
    pred = (fx["pred_bits"], fx["pred_vals"])
    st, cnt = eng.simulate(m["seed"], m["n_traj"], m["n_steps"], traj_begin=m["traj_begin"],
                           step_begin=m["step_begin"], pred=pred, stream=stream)
    assert _without_warps(eng.last_kernel()) == want
    assert np.array_equal(st, fx[f"states_s{stream}"])
    assert np.array_equal(cnt, fx[f"counts_s{stream}"])
